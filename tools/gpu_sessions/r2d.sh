# SBM term kernels: ncu full captures (configs 3, 5) + A/B of sub-groups per row and k=128 unroll
mkdir -p gpurun_out/r2d
N="ncu --set full --import-source on --clock-control none"
timeout 600 $N -k regex:spmm_term_kernel --launch-skip 20 -c 1 -o gpurun_out/r2d/spmm_cfg3 python tools/sweep_spmm.py --config 3 --reps 1 > gpurun_out/r2d/ncu3.log 2>&1
timeout 600 $N -k regex:spmm_term_kernel --launch-skip 25 -c 1 -o gpurun_out/r2d/spmm_cfg5 python tools/sweep_spmm.py --config 5 --reps 1 > gpurun_out/r2d/ncu5.log 2>&1
for C in 3 5; do for R in 1 2; do
  for S in 0 2 4; do
    echo "cfg $C SPED_SUB=$S $(SPED_SUB=$S timeout 300 python tools/sweep_spmm.py --config $C --reps 10 | python -c 'import json,sys; print(" ".join("%.4f" % json.loads(l)["ms_per_term"] for l in sys.stdin if l.startswith("{")))')" >> gpurun_out/r2d/ab_sub.log
  done
done; done
timeout 900 bash tools/ab_variants.sh 5 2 paper_2207_14589_b200/libsped.so build/var2/lib_W8_K128_U_8_W8_K128_MINB_2.so build/var2/lib_W8_K128_U_2_W8_K128_MINB_4.so build/var2/lib_W8_K128_U_4_W8_K128_MINB_3.so > gpurun_out/r2d/ab_k128.log 2>&1
