# ncu --set full of the packed k=32 update and the k=32 / k=64 Gram (bench_gram), after a plain run of the same command
timeout 300 python tools/bench_gram.py --reps 1 > gpurun_out/r2zu_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"block_update_k32_f2|block_update_v2|gram_tc2_kernel|update_tc128" -c 10 -o gpurun_out/r2zu_gram_update python tools/bench_gram.py --reps 1 > gpurun_out/r2zu_ncu.log 2>&1
