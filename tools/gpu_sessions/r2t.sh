# coalesced column-major fp64 drain of the k = 128 Gram: time, error, parity tests
for L in paper_2207_14589_b200/libsped.so build/var10/lib_split1024.so; do
  echo "== $L" >> gpurun_out/r2t_gram.log
  SPED_LIB=$L timeout 300 python tools/bench_gram.py --reps 20 --only 128 >> gpurun_out/r2t_gram.log 2>&1
done
timeout 900 python -m pytest -q -x tests/test_gpu_solver.py -k "gram or k128 or steps_vs_reference or oja" tests/test_gpu_fullsize.py -k "gram or k128 or steps_vs_reference or oja or exact_apply_and_step and 5" > gpurun_out/r2t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_tests.log
