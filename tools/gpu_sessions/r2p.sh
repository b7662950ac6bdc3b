# launch list of one config-5 exact step (where the Gram + update time goes)
timeout 600 python tools/step_cfg.py 5 3 > gpurun_out/r2p_step5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --cache-control none --clock-control none --csv --log-file gpurun_out/r2p_launches_step5.csv python tools/step_cfg.py 5 2 > gpurun_out/r2p_ncu.log 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "large_nk" > gpurun_out/r2p_large_nk.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_large_nk.log
