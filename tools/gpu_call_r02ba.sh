#!/usr/bin/env bash
# HEAD check after the session restart: the whole -m gpu suite, then the bench line.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/t_ba.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_ba.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ba.json 2> gpurun_out/bench_ba_err.log
echo "bench exit $?" >> gpurun_out/bench_ba_err.log
echo done
