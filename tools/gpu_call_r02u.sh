#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
OZ_PROF=1 timeout 300 python tools/oz_probe.py > gpurun_out/oz_prof.log 2>&1
TCB_OZ_DBG=2 OZ_PROF=1 timeout 300 python tools/oz_probe.py >> gpurun_out/oz_prof.log 2>&1
echo done
