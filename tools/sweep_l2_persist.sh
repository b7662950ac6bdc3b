#!/bin/bash
# persisting-L2 window over the hub prefix: set-aside size x window size
# (HOT_FRACTION of the 126 MB L2), config 4 per-term time
for MB in 0 32 40 48 64; do
  echo "== SPED_L2_PERSIST_MB=$MB"
  SPED_L2_PERSIST_MB=$MB timeout 600 python tools/sweep_spmm.py --config 4 --hot 0.2 0.25 0.3 0.4 --reps 10 | cut -c1-190
done
