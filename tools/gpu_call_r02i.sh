#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_oz.log 2>&1
TCB_OZAKI=0 TL_OUT=gpurun_out/timeline_dmma.json timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_dmma.log 2>&1
timeout 600 python tools/c5_core_stats.py 1e-2 > gpurun_out/c5_core_stats.log 2>&1
echo done
