# final-state check (FFMA2 build): GPU suite, smoke, default bench, reference arm, launch list, ncu of the term kernels + update
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2zp_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2zp_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2zp_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2zp_smoke.log
timeout 900 python bench.py > gpurun_out/r2zp_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2zp_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r2zp_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2zp_bench_ref.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > gpurun_out/r2zp_bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -c 400 --csv --log-file gpurun_out/r2zp_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > gpurun_out/r2zp_ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:"spmm_free_kernel|spmm_chunk_kernel|block_update_k32_f2|gram_tc2_kernel" --launch-skip 65 -c 5 -o gpurun_out/r2zp_step_cfg4 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extra > gpurun_out/r2zp_ncu_full.log 2>&1
