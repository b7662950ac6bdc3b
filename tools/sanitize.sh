#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over the parity tests
# of the riskiest kernels: SpMM hub-chunk tickets, the
# tcgen05 Gram/update mbarrier rings, the grid-resident K7 tag protocol,
# the edge-minibatch sort/sweep and the row-shard build.  Logs -> gpurun_out/sanitize_*.log
O=gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL_MEM="test_long_row_chunk_path or test_apply_all_widths_vs_oracle or test_relabelled_operator_matches_oracle or test_gram_kernels_vs_fp64 or test_block_update_vs_fp64 or test_k128_tensor_core_kernels_small_n or test_persistent_solver_tiny or test_edge_batch_poly_vs_restated_oracle or test_edge_batch_all_terms_sort_equals_per_term or test_device_pcg64_bit_exact or test_row_build_equals_full_build_rows"
FILES="tests/test_gpu_parity.py tests/test_gpu_solver.py tests/test_gpu_shard_build.py"
for tool in memcheck racecheck synccheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
    python -m pytest -q -x -p no:cacheprovider $FILES -k "$SEL_MEM" > $O/sanitize_$tool.log 2>&1
  echo "exit=$?" >> $O/sanitize_$tool.log
done
