#!/bin/bash
# bench_support/libdram_meter.so (CUPTI range profiler; measurement only)
set -e
cd "$(dirname "$0")"
C=/usr/local/cuda/targets/x86_64-linux
[ -d "$C" ] || C=/usr/local/cuda
g++ -O2 -shared -fPIC -std=c++17 -I$C/include dram_meter.cpp -o libdram_meter.so \
  -L$C/lib -lcupti -L/usr/local/cuda/lib64/stubs -lcuda -Wl,-rpath,$C/lib
