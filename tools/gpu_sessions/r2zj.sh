# SpMM instruction diet: packed FMAs (FFMA2), one IMAD.WIDE.U32 per gather address, predicated diagonal skip
V=build/var15
for C in 4 3 5; do
  timeout 1200 bash tools/ab_variants.sh $C 3 $V/lib_base.so $V/lib_f1_fma2.so $V/lib_f3_fma2_u32.so $V/lib_f4_fma2_u32_pred.so > gpurun_out/r2zj_ab_diet_cfg$C.log 2>&1
done
