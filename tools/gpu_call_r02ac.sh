#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 120 python tools/ac_bench.py 1000000 > gpurun_out/ac_bench_ac.log 2>&1
timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_ac.log 2>&1
cp gpurun_out/timeline.json gpurun_out/timeline_ac.json
TCB_TRACE=1 C5_ITERS=2 C5_NO_DEC=1 timeout 400 python tools/c5_once.py 1e-2 > gpurun_out/c5_trace_ac.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exact.py tests/test_gpu_decompress.py tests/test_gpu_configs.py -q -x --timeout 900 > gpurun_out/t_ac.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_ac.log
echo done
