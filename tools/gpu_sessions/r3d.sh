# final build (two lane slices for long rows at k = 32): GPU suite, smoke, default bench, reference arm, launch list, config-3 ncu
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3d_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3d_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r3d_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r3d_smoke.log
timeout 900 python bench.py > gpurun_out/r3d_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r3d_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r3d_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r3d_bench_ref.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > gpurun_out/r3d_bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -c 400 --csv --log-file gpurun_out/r3d_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > gpurun_out/r3d_ncu_launches.log 2>&1
timeout 600 python tools/step_cfg.py 3 2 > gpurun_out/r3d_step3_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:spmm_free_kernel --launch-skip 20 -c 2 -o gpurun_out/r3d_spmm_cfg3 python tools/step_cfg.py 3 2 > gpurun_out/r3d_ncu_cfg3.log 2>&1
