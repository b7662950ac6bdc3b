# gathers without L1 allocation (configs 3 / 4 / 5)
for C in 5 3 4; do
  timeout 900 bash tools/ab_variants.sh $C 3 build/var19/lib_base.so build/var19/lib_noalloc.so > gpurun_out/r2zt_ab_noalloc_cfg$C.log 2>&1
done
