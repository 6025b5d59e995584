#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_ah.log 2>&1
cp gpurun_out/timeline.json gpurun_out/timeline_ah.json
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/t_ah.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_ah.log
echo done
