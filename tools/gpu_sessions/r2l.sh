# in-run DRAM meter check, k-means tests, compute-sanitizer over the riskiest kernels
timeout 600 python bench.py --no-cpu --no-extra --steps 5 --warmup 3 > gpurun_out/r2l_bench_meter.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_bench_meter.log
timeout 900 python -m pytest -q -x tests/test_gpu_solver.py -k "kmeans or cfg1_matches" tests/test_gpu_fullsize.py::test_stochastic_run_solver_sbm > gpurun_out/r2l_kmeans_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_kmeans_tests.log
bash tools/sanitize.sh
