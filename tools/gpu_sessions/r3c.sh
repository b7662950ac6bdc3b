# warp-row segment at k = 32: 4 vs 2 vs 1 lane slices per row
for r in 1 2 3; do
  for S in 4 2 1; do
    ms=$(SPED_LONG_SUB=$S timeout 300 python tools/sweep_spmm.py --config 4 --reps 10 | python -c 'import json,sys; print(" ".join("%.4f" % json.loads(l)["ms_per_term"] for l in sys.stdin if l.startswith("{")))')
    echo "$ms  SPED_LONG_SUB=$S" >> gpurun_out/r3c_long_sub.log
  done
done
