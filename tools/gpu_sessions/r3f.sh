# same-process interleaved A/B of the long-row lane slices (config 4)
timeout 900 python tools/ab_long_sub.py --rounds 6 > gpurun_out/r3f_ab_long_sub.log 2>&1
