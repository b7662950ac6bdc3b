# round-end style verification: smoke, GPU suite, default bench, reference arm, launch list, one full capture
O=gpurun_out/final
mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest -q tests -m gpu -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -c 400 --csv --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:spmm_free_kernel --launch-skip 60 -c 2 -o $O/spmm_free_cfg4 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extra > $O/ncu_full.log 2>&1
