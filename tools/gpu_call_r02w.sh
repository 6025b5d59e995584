#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 120 python tools/ac_bench.py 1000000 > gpurun_out/ac_bench_w.log 2>&1
timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_w.log 2>&1
cp gpurun_out/timeline.json gpurun_out/timeline_w.json
TCB_TRACE=1 C5_ITERS=3 C5_NO_DEC=1 timeout 400 python tools/c5_once.py 1e-2 > gpurun_out/c5_trace_w.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_exact.py tests/test_gpu_parity.py -q -x --timeout 900 > gpurun_out/t_w.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_w.log
echo done
