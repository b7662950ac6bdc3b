# ncu --set full (source-level) of the k = 128 update and the k = 32 Gram / update
mkdir -p gpurun_out/r2u
N="ncu --set full --import-source on --clock-control none"
timeout 900 $N -k regex:"update_tc128" -c 1 -o gpurun_out/r2u/upd128 python tools/bench_gram.py --reps 1 --only 128 > gpurun_out/r2u/ncu1.log 2>&1
timeout 900 $N -k regex:"gram_tc2_kernel|block_update_v2" -c 2 -o gpurun_out/r2u/k32 python tools/bench_gram.py --reps 1 --only 32 > gpurun_out/r2u/ncu2.log 2>&1
