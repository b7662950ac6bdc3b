#!/bin/bash
# DRAM bytes / L2 hit rate of the config-4 term kernels with and without the
# persisting-L2 window over the hub prefix (cache state kept between launches).
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum
for MB in 0 48; do
  SPED_L2_PERSIST_MB=$MB timeout 900 ncu --metrics $M --cache-control none --clock-control none \
    -k regex:spmm -c 150 --csv --log-file gpurun_out/l2p_$MB.csv \
    python tools/sweep_spmm.py --config 4 --hot 0.35 --reps 1 > gpurun_out/l2p_$MB.log 2>&1
done
