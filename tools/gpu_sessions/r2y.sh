# k = 32 SIMT update ring / occupancy variants
for r in 1 2; do for L in paper_2207_14589_b200/libsped.so build/var12/*.so; do
  echo "== $L" >> gpurun_out/r2y_upd32.log
  SPED_LIB=$L timeout 300 python tools/bench_gram.py --reps 20 --only 32 >> gpurun_out/r2y_upd32.log 2>&1
done; done
