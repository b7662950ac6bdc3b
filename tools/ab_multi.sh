#!/bin/bash
# interleaved A/B of several library builds on one config's SpMM (2 rounds)
# usage: tools/ab_multi.sh <config> <lib>...
C=$1; shift
for r in 1 2; do
  for L in "$@"; do
    echo "== $L"
    SPED_LIB=$L timeout 300 python tools/sweep_spmm.py --config $C --hot 0.3 --reps 10 | cut -c1-190
  done
done
