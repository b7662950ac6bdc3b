# ncu of the hub sweep kernel (config 4)
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:hub_sweep_kernel --launch-skip 3 -c 1 -o gpurun_out/r2zg_hub_sweep python tools/probe_hub_sweep.py --config 4 --reps 3 > gpurun_out/r2zg_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r2zg_ncu.log
