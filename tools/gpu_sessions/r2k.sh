# default bench; launch list (+DRAM bytes); one full capture of the short-row term kernel
timeout 900 python bench.py > gpurun_out/r2k_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2k_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -c 400 --csv --log-file gpurun_out/r2k_launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > gpurun_out/r2k_ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:spmm_free_kernel --launch-skip 60 -c 3 -o gpurun_out/r2k_spmm_free_cfg4 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extra > gpurun_out/r2k_ncu_full.log 2>&1
