# short-row occupancy x gathers in flight after the instruction diet (configs 3, 4)
V=build/var18
for C in 3 4; do
  timeout 1200 bash tools/ab_variants.sh $C 3 $V/lib_base.so $V/lib_FREE_U2_FREE_MINB5.so $V/lib_FREE_U3_FREE_MINB5.so $V/lib_FREE_U4_FREE_MINB5.so > gpurun_out/r2zm_ab_short_occ_cfg$C.log 2>&1
done
