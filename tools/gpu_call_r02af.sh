#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_af.log 2>&1
cp gpurun_out/timeline.json gpurun_out/timeline_af.json
timeout 300 python tools/timeline.py 1e-3 > gpurun_out/timeline_af3.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/t_af.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_af.log
echo done
