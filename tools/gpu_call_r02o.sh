#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 120 python tools/ac_bench.py 1000000 > gpurun_out/ac_bench_o.log 2>&1
timeout 300 python tools/oz_probe.py > gpurun_out/oz_probe.log 2>&1
TCB_OZAKI_LT=1 timeout 300 python tools/oz_probe.py >> gpurun_out/oz_probe.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"oz_mma_kernel" -c 2 \
    -o gpurun_out/ozmma python tools/oz_probe.py > gpurun_out/ncu_oz.log 2>&1
echo done
