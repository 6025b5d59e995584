#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x > gpurun_out/t_oz.log 2>&1
TCB_TRACE=1 C5_ITERS=3 timeout 400 python tools/c5_once.py 1e-2 > gpurun_out/c5_oz.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_exact.py -q -k "c5 or plane or c2 or c3" > gpurun_out/t_cfg_oz.log 2>&1
echo done
