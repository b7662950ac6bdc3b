#!/bin/bash
# One --set full capture per hot kernel of the final build (key metrics are
# summarised with tools/ncu_summary.py into profiles/).
O=gpurun_out/final
mkdir -p $O
N="ncu --set full --import-source on --clock-control none"
timeout 600 $N -k regex:spmm_term_kernel --launch-skip 60 -c 2 -o $O/spmm_cfg4 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extra > $O/log1 2>&1
timeout 600 $N -k regex:spmm_chunk_kernel --launch-skip 30 -c 1 -o $O/chunk_cfg4 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extra > $O/log2 2>&1
timeout 600 $N -k regex:"gram_tc2_kernel|block_update_v2|update_tc128" -c 8 -o $O/gram_update python tools/bench_gram.py --reps 1 > $O/log3 2>&1
timeout 600 $N -k regex:persistent_mueg -c 1 -o $O/k7 python tools/bench_small.py --steps 20 > $O/log4 2>&1
timeout 600 $N -k regex:"batch_row_kernel|records_kernel" -c 2 -o $O/stochastic python tools/sweep_stochastic.py --config 3 --reps 1 > $O/log5 2>&1
