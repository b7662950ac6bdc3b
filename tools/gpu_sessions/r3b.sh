# warp-row segment at k = 32: 4 lane slices (16 lanes per row) vs 8 (a whole warp per row) vs 2
for r in 1 2 3; do
  for S in 4 8 2; do
    ms=$(SPED_LONG_SUB=$S timeout 300 python tools/sweep_spmm.py --config 4 --reps 10 | python -c 'import json,sys; print(" ".join("%.4f" % json.loads(l)["ms_per_term"] for l in sys.stdin if l.startswith("{")))')
    echo "$ms  SPED_LONG_SUB=$S" >> gpurun_out/r3b_long_sub.log
  done
done
