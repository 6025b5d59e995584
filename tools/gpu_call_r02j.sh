#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 300 python tools/timeline.py 1e-2 > gpurun_out/timeline_j.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/t_all_j.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_all_j.log
C5_PROFILE=1 C5_NO_DEC=1 C5_ITERS=2 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"ex_plane_kernel|sc_emit_kernel|ac_range_kernel" -c 4 -o gpurun_out/full_j python tools/c5_once.py 1e-2 \
    > gpurun_out/ncu_full_j.log 2>&1
echo done
