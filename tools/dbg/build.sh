#!/usr/bin/env bash
# Debug harness build: tridiagonalisation phase timings (clock64) from eig.cu.
set -e
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_TRIDIAG_TIMING --expt-relaxed-constexpr \
    tri_timing.cu ../../paper_2107_01384_b200/csrc/eig.cu -o tri_timing
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr \
    tri_timing.cu ../../paper_2107_01384_b200/csrc/eig.cu -o tri_plain
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_TOPK_TIMING --expt-relaxed-constexpr \
    topk_timing.cu ../../paper_2107_01384_b200/csrc/topk.cu -o topk_timing
