# hub rows stored evict_last for the next term; dead hub prefix demoted after each term
L=paper_2207_14589_b200/libsped.so
V=build/var8
timeout 1500 bash tools/ab_variants.sh 4 3 $L $V/lib_HOT_STORE_1.so $V/lib_DEMOTE_1.so $V/lib_HOT_STORE_1_DEMOTE_1.so "SPED_L2_PERSIST_MB=64:$V/lib_HOT_STORE_1_DEMOTE_1.so" "SPED_L2_PERSIST_MB=0:$V/lib_HOT_STORE_1_DEMOTE_1.so" > gpurun_out/r2o_ab_hot_store.log 2>&1
for H in 0.2 0.4 0.55; do
  echo "hot $H: $(SPED_LIB=$V/lib_HOT_STORE_1_DEMOTE_1.so timeout 300 python tools/sweep_spmm.py --config 4 --hot $H --reps 10 | python -c 'import json,sys; print(" ".join("%.4f" % json.loads(l)["ms_per_term"] for l in sys.stdin if l.startswith("{")))')" >> gpurun_out/r2o_hot_sweep.log
done
