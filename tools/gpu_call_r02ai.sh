#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_ai.log 2>&1
cp gpurun_out/timeline.json gpurun_out/timeline_ai.json
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x --timeout 900 > gpurun_out/t_ai.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_ai.log
echo done
