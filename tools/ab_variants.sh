#!/bin/bash
# interleaved A/B/... of library builds (SPED_LIB=) on one config's SpMM apply
# usage: tools/ab_variants.sh <config> <rounds> <lib> [<lib> ...]
#        (a lib may carry env settings: "ENV=val:path/lib.so")
C=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  for spec in "$@"; do
    envs=""; L=$spec
    if [[ "$spec" == *:* ]]; then envs=${spec%%:*}; L=${spec#*:}; fi
    ms=$(env $envs SPED_LIB=$L timeout 300 python tools/sweep_spmm.py --config $C --reps 10 \
         | python -c 'import json,sys; print(" ".join("%.4f" % json.loads(l)["ms_per_term"] for l in sys.stdin if l.startswith("{")))')
    echo "$ms  $spec"
  done
done
