# hub sweep: plan stats, partial sums vs torch, time, apply with the sweep on / off (config 4); parity tests of the reordered paths
timeout 900 python tools/probe_hub_sweep.py --config 4 > gpurun_out/r2zf_hub_sweep_cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/r2zf_hub_sweep_cfg4.log
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "relabel or chunk or widths or full_size" > gpurun_out/r2zf_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2zf_parity.log
