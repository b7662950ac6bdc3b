# after the FFMA2 / address / occupancy changes: GPU suite on the debug-check build and on the release build; sharded bench at one rank
SPED_LIB=build/debug/libsped_debug.so timeout 2400 python -m pytest -q tests -m gpu -p no:cacheprovider > gpurun_out/r2zn_gpu_tests_debugchecks.log 2>&1; echo "rc=$?" >> gpurun_out/r2zn_gpu_tests_debugchecks.log
timeout 1800 python -m pytest -q tests -m gpu -p no:cacheprovider > gpurun_out/r2zn_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2zn_gpu_tests.log
SPED_FORCE_SHARD=1 timeout 900 python bench.py --no-cpu --no-extra --steps 5 --warmup 3 > gpurun_out/r2zn_bench_shard1.log 2>&1; echo "rc=$?" >> gpurun_out/r2zn_bench_shard1.log
