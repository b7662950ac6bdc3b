# long-row / hub-chunk occupancy x gathers-in-flight A/B on config 4 (free kernels)
V=build/var14
timeout 1500 bash tools/ab_variants.sh 4 3 $V/lib_base.so $V/lib_LONG_MIN_BLOCKS6_FREE_LONG_U2_CHUNK_MIN_BLOCKS6.so $V/lib_LONG_MIN_BLOCKS5_FREE_LONG_U3_CHUNK_MIN_BLOCKS5.so $V/lib_LONG_MIN_BLOCKS6_FREE_LONG_U3_CHUNK_MIN_BLOCKS6.so $V/lib_LONG_MIN_BLOCKS8_FREE_LONG_U2_CHUNK_MIN_BLOCKS8.so $V/lib_LONG_MIN_BLOCKS5_FREE_LONG_U4_CHUNK_MIN_BLOCKS5.so > gpurun_out/r2ze_ab_long_occupancy_cfg4.log 2>&1
