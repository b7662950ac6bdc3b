#!/bin/bash
# per-term SpMM timing of configs 4 (taylor, relabelled), 3 and 5 (limit, natural order)
for c in 4 3 5; do
  K=negexp-limit; R=none
  [ $c = 4 ] && K=negexp-taylor && R=auto
  python tools/sweep_spmm.py --config $c --kind $K --reorder $R 2>&1 | cut -c1-170
done
