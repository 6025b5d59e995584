#!/usr/bin/env bash
# Re-entry check of HEAD: GPU suite, smoke, c5 trace (Ozaki default and DMMA), bench line.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/t_all.log 2>&1
echo "pytest exit $?" >> gpurun_out/t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
TCB_TRACE=1 C5_ITERS=3 C5_NO_DEC=1 timeout 400 python tools/c5_once.py 1e-2 > gpurun_out/c5_oz.log 2>&1
TCB_OZAKI=0 TCB_TRACE=1 C5_ITERS=3 C5_NO_DEC=1 timeout 400 python tools/c5_once.py 1e-2 > gpurun_out/c5_dmma.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench_err.log
echo done
