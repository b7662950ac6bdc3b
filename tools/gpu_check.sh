#!/bin/bash
# GPU-box check: gpu tests, default bench, ncu launch list (warm L2: persisting window kept) and one --set full capture of the short-row term kernel

timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -c 400 --csv --log-file gpurun_out/launches_persist.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:spmm_term_kernel --launch-skip 60 -c 1 -o gpurun_out/spmm_short_persist python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extra > gpurun_out/ncu_full.log 2>&1
