# re-entry check after the container was re-created: GPU suite, default bench, and SM<->L2 port metrics of the SBM term kernels
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2zb_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2zb_gpu_tests.log
timeout 600 python bench.py > gpurun_out/r2zb_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2zb_bench.log
M=gpu__time_duration.sum,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_sectors.sum.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,lts__t_bytes.sum.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
for C in 3 5 4; do
  timeout 600 ncu --metrics $M --cache-control none --clock-control none -k regex:"spmm_free_kernel|spmm_chunk_kernel" --launch-skip 20 -c 6 --csv --log-file gpurun_out/r2zb_port_cfg$C.csv python tools/step_cfg.py $C 2 > gpurun_out/r2zb_port_cfg$C.log 2>&1
done
