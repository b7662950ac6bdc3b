# hub sweep: one wave, gathers in flight x occupancy
V=build/var14
timeout 600 python tools/probe_hub_sweep.py --config 4 > gpurun_out/r2zh_sweep_u12_b6.log 2>&1
SPED_SWEEP_WPS=32 SPED_LIB=$V/lib_SWEEP_U32_SWEEP_MINB4.so timeout 600 python tools/probe_hub_sweep.py --config 4 > gpurun_out/r2zh_sweep_u32_b4.log 2>&1
SPED_SWEEP_WPS=40 SPED_LIB=$V/lib_SWEEP_U16_SWEEP_MINB5.so timeout 600 python tools/probe_hub_sweep.py --config 4 > gpurun_out/r2zh_sweep_u16_b5.log 2>&1
SPED_SWEEP_WPS=32 SPED_LIB=$V/lib_SWEEP_U24_SWEEP_MINB4.so timeout 600 python tools/probe_hub_sweep.py --config 4 > gpurun_out/r2zh_sweep_u24_b4.log 2>&1
