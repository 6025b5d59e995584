#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 300 python tools/oz_diag.py > gpurun_out/oz_diag2.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_configs.py -q -k "ozaki or c5 or config" > gpurun_out/t_oz2.log 2>&1
echo done
