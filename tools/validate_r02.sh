#!/usr/bin/env bash
# One GPU call: c5 fixtures (CPU oracle, in the background), the GPU suite,
# a c5 trace, the Ozaki evaluation, then the round's profiles.
set -u
mkdir -p gpurun_out
(timeout 2400 python tests/golden/make_c5_fixtures.py 0.01 > gpurun_out/c5fix1.log 2>&1;
 cp tests/golden/c5_fixtures.json gpurun_out/c5_fixtures.json) &
FIX=$!
timeout 1800 python -m pytest tests -m gpu -q -k "not c5_against" > gpurun_out/t_all.log 2>&1
TCB_TRACE=1 C5_ITERS=2 timeout 300 python tools/c5_once.py 1e-2 > gpurun_out/c5_trace.log 2>&1
timeout 600 python tools/ozaki_eval.py 4 5 6 7 > gpurun_out/ozaki.log 2>&1
wait $FIX
bash tools/profile_round.sh
