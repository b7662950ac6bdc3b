# no diagonal gather (VM 2: exact; VM 1: diagonal from the own row, A/B)
L=paper_2207_14589_b200/libsped.so
for C in 4 3 5; do
  timeout 900 bash tools/ab_variants.sh $C 3 build/var13/lib_base.so $L build/var13/lib_diag_epi.so > gpurun_out/r2za_ab_diag_cfg$C.log 2>&1
done
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "not config2 and not stochastic_run" > gpurun_out/r2za_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2za_parity.log
SPED_LIB=build/var13/lib_diag_epi.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "not config2 and not stochastic_run" > gpurun_out/r2za_parity_diag_epi.log 2>&1; echo "rc=$?" >> gpurun_out/r2za_parity_diag_epi.log
