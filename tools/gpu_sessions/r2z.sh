# hub window vs hints on a power-law gather stream (probe), with ncu DRAM bytes
./tools/probe/hub_window > gpurun_out/r2z_hub_window.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/r2z_hub_window_ncu.csv ./tools/probe/hub_window > /dev/null 2>&1
