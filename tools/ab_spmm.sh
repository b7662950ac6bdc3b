#!/bin/bash
# interleaved A/B of two library builds on the config-4 SpMM (3 rounds)
# usage: tools/ab_spmm.sh <libA.so> <libB.so> [config]
A=$1; B=$2; C=${3:-4}
for r in 1 2 3; do
  for L in $A $B; do
    echo "== $L"
    SPED_LIB=$L timeout 300 python tools/sweep_spmm.py --config $C --hot 0.3 --reps 10 | cut -c1-190
  done
done
