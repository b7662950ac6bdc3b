# transposed-accumulator k = 128 update: time and error
for L in paper_2207_14589_b200/libsped.so build/var10/lib_upd_trans.so; do
  echo "== $L" >> gpurun_out/r2v_upd.log
  SPED_LIB=$L timeout 300 python tools/bench_gram.py --reps 20 --only 128 >> gpurun_out/r2v_upd.log 2>&1
done
SPED_LIB=build/var10/lib_upd_trans.so timeout 900 python -m pytest -q -x tests/test_gpu_solver.py -k "k128 or block_update or steps_vs_reference or oja" > gpurun_out/r2v_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_tests.log
