# epilogue prefetch A/B (EPI_PREFETCH=1: x row; 2: x and own row) on configs 3/4/5
for C in 3 4 5; do
  timeout 900 bash tools/ab_variants.sh $C 3 build/var14/lib_base.so build/var14/lib_EPI_PREFETCH1.so build/var14/lib_EPI_PREFETCH2.so > gpurun_out/r2zd_ab_epi_prefetch_cfg$C.log 2>&1
done
