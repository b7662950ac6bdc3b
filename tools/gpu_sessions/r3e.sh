# bench with the DRAM-meter retry: default line (for profiles) and two short runs
timeout 900 python bench.py > gpurun_out/r3e_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r3e_bench.log
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-extra > gpurun_out/r3e_bench_short_$i.log 2>&1; echo "rc=$?" >> gpurun_out/r3e_bench_short_$i.log; done
