#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
TCB_TRACE=1 C5_ITERS=3 C5_NO_DEC=1 timeout 300 python tools/c5_once.py 1e-2 > gpurun_out/c5_trace2.log 2>&1
TCB_TRACE=1 timeout 300 python tools/compress_once.py --config c2 --re 1e-4 --warmup 3 --steps 2 > gpurun_out/c2_trace.log 2>&1
(timeout 2700 python tests/golden/make_c5_fixtures.py 0.001 > gpurun_out/c5fix2.log 2>&1;
 cp tests/golden/c5_fixtures.json gpurun_out/c5_fixtures.json) &
FIX=$!
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -k "eig or early or c5 or config" > gpurun_out/t_sub.log 2>&1
C5_PROFILE=1 C5_NO_DEC=1 C5_ITERS=2 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/launches2.csv python tools/c5_once.py 1e-2 > gpurun_out/ncu_c5b.log 2>&1
C5_PROFILE=1 C5_NO_DEC=1 C5_ITERS=2 timeout 900 ncu --profile-from-start off --set full --import-source on \
    --clock-control none -k regex:"ex_plane_kernel|sc_emit_kernel|tridiag_coop_smem" -c 4 -o gpurun_out/full_enc \
    python tools/c5_once.py 1e-2 > gpurun_out/ncu_enc.log 2>&1
wait $FIX
echo done
