#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 120 python tools/ac_bench.py 1000000 > gpurun_out/ac_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"ac_range_kernel" -c 1 \
    -o gpurun_out/ac_range python tools/ac_bench.py 1000000 > gpurun_out/ncu_ac.log 2>&1
echo done
