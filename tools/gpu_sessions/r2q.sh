# programmatic dependent launch of the term kernels (SPED_PDL=1): smoke, A/B, parity
L=paper_2207_14589_b200/libsped.so
SPED_PDL=1 timeout 300 python tools/sweep_spmm.py --config 4 --reps 10 > gpurun_out/r2q_pdl_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_pdl_smoke.log
if grep -q "rc=0" gpurun_out/r2q_pdl_smoke.log; then
  for C in 4 3 5; do
    timeout 900 bash tools/ab_variants.sh $C 3 "SPED_PDL=0:$L" "SPED_PDL=1:$L" > gpurun_out/r2q_ab_pdl_cfg$C.log 2>&1
  done
  SPED_PDL=1 timeout 1500 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_solver.py tests/test_gpu_shard_build.py tests/test_gpu_fullsize.py -k "not config2 and not stochastic_run" > gpurun_out/r2q_pdl_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_pdl_parity.log
fi
