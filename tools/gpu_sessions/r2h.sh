# shuffle-free kernel tuning (U x min blocks) and parity with it on
L=paper_2207_14589_b200/libsped.so
V=build/var6
for C in 3 5 4; do
  timeout 1500 bash tools/ab_variants.sh $C 2 "SPED_FREE=1:$L" "SPED_FREE=1:$V/lib_FREE_U_2_FREE_MINB_5.so" "SPED_FREE=1:$V/lib_FREE_U_3_FREE_MINB_5.so" "SPED_FREE=1:$V/lib_FREE_U_3_FREE_MINB_6.so" "SPED_FREE=1:$V/lib_FREE_U_4_FREE_MINB_5.so" > gpurun_out/r2h_ab_free_tune_cfg$C.log 2>&1
done
SPED_FREE=1 timeout 900 python -m pytest -q -x tests/test_gpu_fullsize.py -k "exact_apply" tests/test_gpu_parity.py tests/test_gpu_distributed.py tests/test_gpu_shard_build.py > gpurun_out/r2h_free_parity.log 2>&1
