# free kernels everywhere (short rows, warp rows, chunks) vs shuffle kernels; full GPU suite with them on
L=paper_2207_14589_b200/libsped.so
for C in 4 3 5; do
  timeout 900 bash tools/ab_variants.sh $C 3 "SPED_FREE=0:$L" "SPED_FREE=1:$L" > gpurun_out/r2i_ab_free_all_cfg$C.log 2>&1
done
SPED_FREE=1 timeout 1800 python -m pytest -q -x tests -m gpu > gpurun_out/r2i_gpu_tests_free.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_gpu_tests_free.log
