#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x --timeout 300 > gpurun_out/t_oz_n.log 2>&1
rc=$?
echo "pytest exit $rc" >> gpurun_out/t_oz_n.log
if [ $rc -ne 0 ]; then echo done; exit 0; fi
timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_n.log 2>&1
cp gpurun_out/timeline.json gpurun_out/timeline_n.json
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/t_all_n.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_all_n.log
echo done
