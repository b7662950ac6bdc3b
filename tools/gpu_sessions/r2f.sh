# A/B: 128-bit gathers (SPED_VEC=4) on the SBM configs; L2 hint variants on config 4
L=paper_2207_14589_b200/libsped.so
for C in 3 5; do
  timeout 900 bash tools/ab_variants.sh $C 2 "SPED_VEC=8:$L" "SPED_VEC=4:$L" > gpurun_out/r2f_ab_vec_cfg$C.log 2>&1
done
timeout 900 bash tools/ab_variants.sh 4 3 "SPED_VEC=8:$L" "SPED_VEC=8:build/var4/lib_hints1.so" "SPED_VEC=8:build/var4/lib_hints2.so" > gpurun_out/r2f_ab_hints_cfg4.log 2>&1
