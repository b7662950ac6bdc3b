# ncu --set full of the k = 128 mu-EG Gram and update (source-level stalls)
mkdir -p gpurun_out/r2r
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gram_tc2_kernel|update_tc128" -c 2 -o gpurun_out/r2r/gram_update_k128 python tools/bench_gram.py --reps 1 --only 128 > gpurun_out/r2r/ncu.log 2>&1
timeout 300 python tools/bench_gram.py --reps 20 > gpurun_out/r2r/bench_gram.log 2>&1
