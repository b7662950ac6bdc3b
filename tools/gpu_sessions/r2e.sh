# shared-memory ring SpMM (short rows): A/B vs register gathers, and parity with the ring on
L=paper_2207_14589_b200/libsped.so
for C in 3 5 4; do
  timeout 1200 bash tools/ab_variants.sh $C 2 "SPED_RING=0:$L" "SPED_RING=1:$L" "SPED_RING=1:build/var3/lib_RING_D_3_RING_MIN_BLOCKS_8.so" "SPED_RING=1:build/var3/lib_RING_D_6_RING_MIN_BLOCKS_4.so" "SPED_RING=1:build/var3/lib_RING_D_2_RING_MIN_BLOCKS_8.so" > gpurun_out/r2e_ab_ring_cfg$C.log 2>&1
done
SPED_RING=1 timeout 900 python -m pytest -q -x tests/test_gpu_fullsize.py -k "exact_apply" tests/test_gpu_parity.py > gpurun_out/r2e_ring_parity.log 2>&1
