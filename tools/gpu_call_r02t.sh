#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x --timeout 300 > gpurun_out/t_oz_t.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_oz_t.log
for d in 0 1 2; do echo "dbg=$d" >> gpurun_out/oz_dbg_t.log; TCB_OZ_DBG=$d timeout 300 python tools/oz_probe.py >> gpurun_out/oz_dbg_t.log 2>&1; done
echo done
