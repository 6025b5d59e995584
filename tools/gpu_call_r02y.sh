#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_y.log 2>&1
bash tools/profile_round.sh
echo done
