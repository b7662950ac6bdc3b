# stochastic sweep: unconditional (clamped) record / gather loads, opaque lane base, occupancy
V=build/var22
for r in 1 2 3; do
  for L in $V/lib_base.so $V/lib_uncond_b8.so $V/lib_uncond_opaque_b8.so $V/lib_uncond_opaque_b6.so $V/lib_uncond_opaque_b6_u3.so; do
    for C in 3 5; do
      echo "== $L cfg $C" >> gpurun_out/r2zy_sto.log
      SPED_LIB=$L timeout 300 python tools/sweep_stochastic.py --config $C --reps 10 >> gpurun_out/r2zy_sto.log 2>&1
    done
  done
done
SPED_LIB=$V/lib_uncond_opaque_b8.so timeout 900 python -m pytest -q -x tests/test_gpu_solver.py tests/test_gpu_fullsize.py -k "batch or stochastic or sto" -p no:cacheprovider > gpurun_out/r2zy_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2zy_tests.log
