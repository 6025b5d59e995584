#!/usr/bin/env bash
# Row-slab Ozaki upload: bitwise tests, then the bench's e2e.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "upload" > gpurun_out/t_bb.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_bb.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/bench_bb.json 2> gpurun_out/bench_bb_err.log
echo "bench exit $?" >> gpurun_out/bench_bb_err.log
TCB_PLAIN_UPLOAD=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/bench_bb_plain.json 2>> gpurun_out/bench_bb_err.log
echo done
