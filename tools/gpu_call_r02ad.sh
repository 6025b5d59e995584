#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_ad.log 2>&1
cp gpurun_out/timeline.json gpurun_out/timeline_ad.json
OZ_PROF=1 timeout 300 python tools/oz_probe.py 2>&1 | grep -v Warn > gpurun_out/oz_ad.log
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/t_ad.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_ad.log
echo done
