# after the float2 alignment guard of the packed update: solver + property tests, update timing
timeout 900 python -m pytest -q -x tests/test_gpu_solver.py tests/test_gpu_properties.py -p no:cacheprovider > gpurun_out/r2zq_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2zq_tests.log
timeout 300 python tools/bench_gram.py --only 32 --reps 20 > gpurun_out/r2zq_update_k32.log 2>&1
