# L2 gather ceiling; interleaved-scratch persisting window sweep (config 4)
./tools/probe/l2_gather > gpurun_out/r2c_l2_gather.log 2>&1
for I in 0 1; do for MB in 40 64 80 96; do
  echo "== SPED_INTERLEAVE=$I SPED_L2_PERSIST_MB=$MB" >> gpurun_out/r2c_window_sweep.log
  SPED_INTERLEAVE=$I SPED_L2_PERSIST_MB=$MB timeout 300 python tools/sweep_spmm.py --config 4 --hot 0.2 0.3 0.4 0.55 --reps 10 2>&1 \
    | python -c 'import json,sys
for l in sys.stdin:
    if l.startswith("{"): d=json.loads(l); print("hot %.2f  %.4f ms/term" % (d["hot_fraction"], d["ms_per_term"]))
    else: print(l.rstrip())' >> gpurun_out/r2c_window_sweep.log
done; done
SPED_INTERLEAVE=1 SPED_L2_PERSIST_MB=80 timeout 600 python -m pytest -q -x tests/test_gpu_fullsize.py -k "exact_apply_and_step and 4" > gpurun_out/r2c_inter_parity.log 2>&1
