#!/bin/bash
for r in 1 2; do
  for sp in 0 1 2 4; do
    echo "== spare$sp"; SPED_STO_SPARE=$sp SPED_LIB=build/variants/sto_new.so python tools/sweep_stochastic.py --config 3 --reps 10
  done
  echo "== nooverlap"; SPED_STO_OVERLAP=0 SPED_LIB=build/variants/sto_new.so python tools/sweep_stochastic.py --config 3 --reps 10
  echo "== old"; SPED_LIB=build/variants/sto_old.so python tools/sweep_stochastic.py --config 3 --reps 10
done
