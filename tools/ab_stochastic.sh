#!/bin/bash
# Stochastic apply per term for several library builds, interleaved
# usage: tools/ab_stochastic.sh <rounds> <lib> [<lib> ...]
R=$1; shift
for r in $(seq 1 $R); do
  for L in "$@"; do
    for c in 3 5; do
      out=$(SPED_LIB=$L timeout 300 python tools/sweep_stochastic.py --config $c --reps 10 | \
            python -c 'import json,sys
for l in sys.stdin:
    if l.startswith("{"):
        d = json.loads(l); print("%.4f ms/term  draw %.3f ms  %s" % (d["ms_per_term"], d["draw_ms_per_apply"], d["out_hash"]))')
      echo "cfg$c $out  $L"
    done
  done
done
