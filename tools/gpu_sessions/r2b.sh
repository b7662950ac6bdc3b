# round-2 probes: gather granularity, config-4 panel-width proxy + panel mode, SBM MLP variants
./tools/probe/gather_bw > gpurun_out/r2b_gather_bw.log 2>&1
timeout 600 python tools/sweep_spmm.py --config 4 --k 8 16 32 --reps 10 > gpurun_out/r2b_k_sweep_cfg4.log 2>&1
for P in 0 16 8 0 16 8; do
  SPED_PANEL_K=$P timeout 600 python tools/sweep_spmm.py --config 4 --reps 10 2>&1 | sed "s/^/panel=$P /" >> gpurun_out/r2b_panel_cfg4.log
done
SPED_PANEL_K=16 timeout 600 python -m pytest -q -x tests/test_gpu_fullsize.py -k "exact_apply_and_step and 4" > gpurun_out/r2b_panel_parity.log 2>&1
for C in 3 5; do
  timeout 900 bash tools/ab_variants.sh $C 3 paper_2207_14589_b200/libsped.so build/var/lib_W8_U_2.so build/var/lib_W8_U_2_TERM_MIN_BLOCKS_W8_6.so build/var/lib_W8_U_4_TERM_MIN_BLOCKS_W8_4.so > gpurun_out/r2b_ab_mlp_cfg$C.log 2>&1
done
