# k = 128 Gram ring depth after the drain fix
for L in paper_2207_14589_b200/libsped.so build/var11/*.so; do
  echo "== $L" >> gpurun_out/r2x_gram.log
  SPED_LIB=$L timeout 300 python tools/bench_gram.py --reps 20 --only 128 >> gpurun_out/r2x_gram.log 2>&1
done
