#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
run() { TCB_TRACE=1 C5_ITERS=3 C5_NO_DEC=1 timeout 300 python tools/c5_once.py 1e-2 > gpurun_out/$1 2>&1; }
run c5_default.log
TCB_NO_EARLY_PLANES=1 run c5_noearly.log
TCB_NO_SUM_OVERLAP=1 run c5_nooverlap.log
TCB_NO_EARLY_PLANES=1 TCB_NO_SUM_OVERLAP=1 run c5_neither.log
TCB_TRACE=1 timeout 300 python tools/compress_once.py --config c2 --re 1e-4 --warmup 3 --steps 2 > gpurun_out/c2_trace4.log 2>&1
timeout 300 python tools/ozaki_eval.py 5 > gpurun_out/ozaki2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "not c5_against" > gpurun_out/t_all4.log 2>&1
echo done
