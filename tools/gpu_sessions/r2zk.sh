# packed-FMA k=32 update (UPD_F2) vs the lane-per-column update; combined SpMM diet build vs the committed base; parity
for r in 1 2 3; do
  for L in build/var16/lib_upd_f2_0.so build/var16/lib_new.so; do
    echo "== $L" >> gpurun_out/r2zk_update_k32.log
    SPED_LIB=$L timeout 300 python tools/bench_gram.py --only 32 --reps 20 >> gpurun_out/r2zk_update_k32.log 2>&1
  done
done
timeout 900 python -m pytest -q -x tests/test_gpu_solver.py tests/test_gpu_parity.py > gpurun_out/r2zk_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2zk_parity.log
for C in 4 3 5; do
  timeout 900 bash tools/ab_variants.sh $C 3 build/var15/lib_base.so build/var16/lib_new.so > gpurun_out/r2zk_ab_diet_final_cfg$C.log 2>&1
done
