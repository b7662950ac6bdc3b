# lean short-row kernel: gathers in flight U = 2 / 3 / 4 at 6 blocks (config 4); final lib vs previous on configs 3 / 5
V=build/var21
timeout 1200 bash tools/ab_variants.sh 4 3 $V/lib_base.so $V/lib_FREE_U3.so $V/lib_FREE_U4.so > gpurun_out/r2zw_ab_u_cfg4.log 2>&1
for C in 3 5; do
  timeout 600 bash tools/ab_variants.sh $C 3 build/var20/lib_base.so $V/lib_base.so > gpurun_out/r2zw_ab_final_cfg$C.log 2>&1
done
