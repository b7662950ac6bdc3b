#!/bin/bash
# Stochastic apply per term: one sort for all terms vs per-term sorts (same library)
for r in 1 2; do
  for c in 3 5; do
    for A in 1 0; do
      echo "== allterms=$A cfg$c"
      SPED_STO_ALLTERMS=$A timeout 300 python tools/sweep_stochastic.py --config $c --reps 10
    done
  done
done
