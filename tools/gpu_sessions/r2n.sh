# stochastic sweep variants; config-4 long-row variants; ncu of the free kernel at configs 3 / 5
L=paper_2207_14589_b200/libsped.so
V=build/var8
timeout 1500 bash tools/ab_stochastic.sh 2 $L $V/lib_sto_rows.so $V/lib_STO_U_4_STO_MINB_6.so $V/lib_STO_U_3_STO_MINB_6.so $V/lib_STO_U_1_STO_MINB_8.so > gpurun_out/r2n_ab_sto.log 2>&1
timeout 900 bash tools/ab_variants.sh 4 3 $L $V/lib_chunk_w8.so $V/lib_chunk_mb6.so $V/lib_long_mb6.so > gpurun_out/r2n_ab_cfg4_long.log 2>&1
mkdir -p gpurun_out/r2n
N="ncu --set full --import-source on --clock-control none"
timeout 600 $N -k regex:spmm_free_kernel --launch-skip 20 -c 1 -o gpurun_out/r2n/free_cfg3 python tools/sweep_spmm.py --config 3 --reps 1 > gpurun_out/r2n/ncu3.log 2>&1
timeout 600 $N -k regex:spmm_free_kernel --launch-skip 25 -c 1 -o gpurun_out/r2n/free_cfg5 python tools/sweep_spmm.py --config 5 --reps 1 > gpurun_out/r2n/ncu5.log 2>&1
