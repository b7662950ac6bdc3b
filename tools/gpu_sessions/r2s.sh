# k = 128 Gram pipeline depth / drain interval variants (time and error)
for L in paper_2207_14589_b200/libsped.so build/var9/*.so; do
  echo "== $L" >> gpurun_out/r2s_gram_variants.log
  SPED_LIB=$L timeout 300 python tools/bench_gram.py --reps 20 --only 128 >> gpurun_out/r2s_gram_variants.log 2>&1
done
