#!/bin/bash
# all-terms sort: split into 24-bit-key groups vs one sort (same library)
for r in 1 2; do
  for c in 3 5; do
    for S in 1 0; do
      echo "== split=$S cfg$c"
      SPED_STO_SPLIT=$S timeout 300 python tools/sweep_stochastic.py --config $c --reps 10
    done
  done
done
