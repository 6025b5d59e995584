#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 300 python tools/oz_probe.py > gpurun_out/oz_probe_q.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x --timeout 300 > gpurun_out/t_oz_q.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_oz_q.log
timeout 120 python tools/ac_bench.py 1000000 > gpurun_out/ac_bench_q.log 2>&1
echo done
