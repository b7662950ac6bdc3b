#!/bin/bash
# K7 per-step time (configs 1-2) for several library builds, interleaved
for r in 1 2; do
  for L in "$@"; do
    echo "== $L"
    SPED_LIB=$L timeout 300 python tools/bench_small.py --steps 500
  done
done
