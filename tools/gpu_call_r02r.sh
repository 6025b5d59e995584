#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
for d in 0 1 2; do echo "dbg=$d" >> gpurun_out/oz_dbg.log; TCB_OZ_DBG=$d timeout 300 python tools/oz_probe.py >> gpurun_out/oz_dbg.log 2>&1; done
echo done
