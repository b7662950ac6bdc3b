# persisting set-aside x hub-window fraction with the final kernels (config 4)
for MB in 32 40 48 60; do
  SPED_L2_PERSIST_MB=$MB timeout 600 python tools/sweep_spmm.py --config 4 --reps 10 --hot 0.2 0.25 0.3 0.35 0.45 > gpurun_out/r2zz_l2_${MB}.log 2>&1
done
