# lane base / row stride kept opaque (no per-gather rematerialisation): A/B on configs 3 / 4 / 5, parity
for C in 3 4 5; do
  timeout 900 bash tools/ab_variants.sh $C 3 build/var20/lib_base.so build/var20/lib_opaque.so > gpurun_out/r2zv_ab_opaque_cfg$C.log 2>&1
done
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "not config2 and not stochastic_run" -p no:cacheprovider > gpurun_out/r2zv_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2zv_parity.log
