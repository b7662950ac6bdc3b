#!/bin/bash
# Stochastic apply per term for several library builds, interleaved
for r in 1 2; do
  for L in "$@"; do
    for c in 3 5; do
      echo "== $L cfg$c"
      SPED_LIB=$L timeout 300 python tools/sweep_stochastic.py --config $c --reps 10
    done
  done
done
