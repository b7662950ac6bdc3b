# shuffle-free short-row kernel A/B; exchange model
L=paper_2207_14589_b200/libsped.so
for C in 3 5 4; do
  timeout 1200 bash tools/ab_variants.sh $C 2 "SPED_FREE=0:$L" "SPED_FREE=1:$L" "SPED_FREE=1:build/var5/lib_FREE_U_1_FREE_MINB_8.so" "SPED_FREE=1:build/var5/lib_FREE_U_2_FREE_MINB_8.so" "SPED_FREE=1:build/var5/lib_FREE_U_4_FREE_MINB_4.so" > gpurun_out/r2g_ab_free_cfg$C.log 2>&1
done
timeout 1200 python tools/exchange_model.py > gpurun_out/r2g_exchange_model.jsonl 2> gpurun_out/r2g_exchange_model.err
