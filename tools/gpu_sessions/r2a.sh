nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/r2a_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2a_gpu_tests.log
timeout 600 python bench.py > gpurun_out/r2a_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2a_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2a_bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/r2a_bench_ref.log
