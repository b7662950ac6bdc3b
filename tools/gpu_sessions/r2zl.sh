# FFMA2 in f4_fma (stochastic sweep, row update kernels) and the k=64 update; A/B against the previous build
for r in 1 2 3; do
  for L in build/var16/lib_new.so build/var17/lib_new2.so; do
    echo "== $L" >> gpurun_out/r2zl_update_k64.log
    SPED_LIB=$L timeout 300 python tools/bench_gram.py --only 64 --reps 50 >> gpurun_out/r2zl_update_k64.log 2>&1
    for C in 3 5; do
      echo "== $L cfg $C" >> gpurun_out/r2zl_sto.log
      SPED_LIB=$L timeout 300 python tools/sweep_stochastic.py --config $C --reps 10 >> gpurun_out/r2zl_sto.log 2>&1
    done
  done
done
timeout 900 python -m pytest -q -x tests/test_gpu_solver.py tests/test_gpu_fullsize.py -k "not config2" > gpurun_out/r2zl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2zl_tests.log
