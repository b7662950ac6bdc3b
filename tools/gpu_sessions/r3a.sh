# last flakiness check of the final build: the GPU suite on the debug-check build and twice on the release build
SPED_LIB=build/debug/libsped_debug.so timeout 2400 python -m pytest -q tests -m gpu -p no:cacheprovider > gpurun_out/r3a_gpu_tests_debugchecks.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_gpu_tests_debugchecks.log
for i in 1 2; do timeout 1800 python -m pytest -q tests -m gpu -p no:cacheprovider > gpurun_out/r3a_gpu_tests_$i.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_gpu_tests_$i.log; done
