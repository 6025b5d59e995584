#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x --timeout 300 > gpurun_out/t_aa.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_aa.log
OZ_PROF=1 timeout 300 python tools/oz_probe.py 2>&1 | grep -v Warn > gpurun_out/oz_aa.log
echo done
