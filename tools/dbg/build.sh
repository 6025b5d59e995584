#!/usr/bin/env bash
# Debug harness build: tridiagonalisation and top-p phase timings (clock64).
set -e
cd "$(dirname "$0")"
rm -f tri_timing tri_plain topk_timing
CSRC=../../paper_2107_01384_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr"
nvcc $F -DTCB_TOPK_TIMING topk_timing.cu $CSRC/topk.cu -o topk_timing
nvcc $F -DTCB_TRIDIAG_TIMING tri_timing.cu $CSRC/eig.cu $CSRC/topk.cu -o tri_timing
nvcc $F -lineinfo tri_timing.cu $CSRC/eig.cu $CSRC/topk.cu -o tri_plain
