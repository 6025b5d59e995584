#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
for d in 0 3; do echo "dbg=$d" >> gpurun_out/oz_dbg_z.log; TCB_OZ_DBG=$d OZ_PROF=1 timeout 300 python tools/oz_probe.py 2>&1 | grep -v Warn >> gpurun_out/oz_dbg_z.log; done
timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_z.log 2>&1
cp gpurun_out/timeline.json gpurun_out/timeline_z.json
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exact.py tests/test_gpu_decompress.py -q -x --timeout 900 > gpurun_out/t_z.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_z.log
echo done
