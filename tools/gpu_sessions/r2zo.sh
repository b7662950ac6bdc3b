# derandomized property tests (3 runs: same examples), then the full suite
for i in 1 2 3; do timeout 600 python -m pytest -q tests/test_gpu_properties.py -p no:cacheprovider > gpurun_out/r2zo_props_$i.log 2>&1; echo "rc=$?" >> gpurun_out/r2zo_props_$i.log; done
timeout 1800 python -m pytest -q tests -m gpu -x -p no:cacheprovider > gpurun_out/r2zo_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2zo_gpu_tests.log
