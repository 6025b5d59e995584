#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 120 python tools/ac_bench.py 1000000 > gpurun_out/ac_bench_m.log 2>&1
timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_m.log 2>&1
cp gpurun_out/timeline.json gpurun_out/timeline_m.json
TCB_EARLY_PLANES=1 timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_m_early.log 2>&1
cp gpurun_out/timeline.json gpurun_out/timeline_m_early.json
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -k "not c5" > gpurun_out/t_m.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_m.log
echo done
