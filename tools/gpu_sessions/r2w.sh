# k = 128 update: coalesced converter loads (same layout, same MMAs)
for L in paper_2207_14589_b200/libsped.so build/var10/lib_upd_coal.so paper_2207_14589_b200/libsped.so build/var10/lib_upd_coal.so; do
  echo "== $L" >> gpurun_out/r2w_upd.log
  SPED_LIB=$L timeout 300 python tools/bench_gram.py --reps 20 --only 128 >> gpurun_out/r2w_upd.log 2>&1
done
