#!/bin/bash
# row sweep: lane-group hsum + group-0-only row loads (sto_lean) vs HEAD (sto_head)
for r in 1 2 3; do
  for L in build/variants/sto_head.so build/variants/sto_lean.so; do
    for c in 3 5; do
      echo "== $L cfg$c"
      SPED_LIB=$L timeout 300 python tools/sweep_stochastic.py --config $c --reps 20
    done
  done
done
