#!/usr/bin/env bash
# compute-sanitizer over one compress + decompress per code path (run on the GPU
# box via gpurun): memcheck everywhere, racecheck + initcheck on the small case.
# Log: gpurun_out/sanitize.log (summary lines only).
set -u
mkdir -p gpurun_out
LOG=gpurun_out/sanitize.log
: > $LOG
run() {  # tool, then the case's arguments
    local tool=$1; shift
    echo "== $tool: $*" >> $LOG
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 5 \
        python tools/sanitize_case.py "$@" > gpurun_out/san_tmp.log 2>&1
    echo "exit $?" >> $LOG
    grep -E "^shape|ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Uninitialized|hazard|AssertionError|Error" gpurun_out/san_tmp.log | head -12 >> $LOG
}
run memcheck 64 64 64 1e-3 float32 sin            # c1: certified top-p eigensolver, DMMA Gram/TTM
run memcheck 200 12 10 1e-6 float64 sin_decay     # thin-SVD branch (rows > cols)
run memcheck 300 48 40 1e-3 float32 blobs         # full eigensolver, DSMEM-cluster tridiagonalisation
run memcheck 700 40 36 1e-3 float32 blobs         # whole-GPU cooperative tridiagonalisation
run memcheck 256 512 512 1e-3 float32 blobs       # Ozaki digits + tcgen05 Gram and TTM
run racecheck 64 64 64 1e-3 float32 sin
run initcheck 64 64 64 1e-3 float32 sin
rm -f gpurun_out/san_tmp.log
cat $LOG
