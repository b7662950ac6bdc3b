# config-4 variants of the free kernels; default bench; launch list (+DRAM bytes); one full capture
L=paper_2207_14589_b200/libsped.so
V=build/var7
timeout 900 bash tools/ab_variants.sh 4 3 "$L" "$V/lib_idx_ef.so" "$V/lib_long_u8.so" "$V/lib_long_u2.so" > gpurun_out/r2j_ab_cfg4.log 2>&1
timeout 900 python bench.py > gpurun_out/r2j_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -c 400 --csv --log-file gpurun_out/r2j_launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > gpurun_out/r2j_ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:spmm_free_kernel --launch-skip 60 -c 3 -o gpurun_out/r2j_spmm_free_cfg4 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extra > gpurun_out/r2j_ncu_full.log 2>&1
