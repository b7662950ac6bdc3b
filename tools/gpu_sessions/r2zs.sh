# launch lists: one exact step of config 5 (Gram / reduce / coefficients / update at k = 128) and the stochastic apply of config 3
timeout 300 python tools/step_cfg.py 5 2 > gpurun_out/r2zs_step5_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --launch-skip 100 -c 200 --csv --log-file gpurun_out/r2zs_launches_cfg5.csv python tools/step_cfg.py 5 2 > gpurun_out/r2zs_ncu5.log 2>&1
timeout 300 python tools/sweep_stochastic.py --config 3 --reps 2 > gpurun_out/r2zs_sto3_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --launch-skip 150 -c 200 --csv --log-file gpurun_out/r2zs_launches_sto3.csv python tools/sweep_stochastic.py --config 3 --reps 2 > gpurun_out/r2zs_ncu_sto3.log 2>&1
