// Core quantisation helpers and the factor (Householder) codec kernels.
#pragma once

#include "common.cuh"

namespace tcb {

// vectorize::OrderMap::build on the device (flat position of each coefficient);
// empty for the lexicographic method (identity)
DevBuf<u64> order_map_device(int method, const std::vector<u64>& shape, cudaStream_t s);
// per-axis "all insignificant" bitmaps, concatenated over axes (core_codec.cpp:510-523)
std::vector<u8> dead_slices(const u64* dec, const std::vector<u64>& shape, cudaStream_t s,
                            const u64* order = nullptr);
// neg ^= parity of factor column flips along each storage axis (pipeline.cpp:161-175)
void sign_fold(u8* neg, const std::vector<u64>& shape, const std::vector<signed char>& flips_by_axis,
               cudaStream_t s, const u64* order = nullptr);

// ---- factor.cu (factor_codec.cpp:23-244)
// max |U_live^T U_live - I| (the orthonormality guard of factorize), computed in T
double orth_deviation(const double* U, u64 n, u64 r, const std::vector<u64>& live, bool as_float, cudaStream_t s);
// Householder reflectors of the live columns: V (column-major n x rl), flips[rl]
void householder(const double* U, u64 n, u64 r, const std::vector<u64>& live, double* V, signed char* flips_host,
                 cudaStream_t s);
// weighted reflector stream: st[s] = V(i,j) * scale_j for j < rl, i > j (column-major)
void reflector_stream(const double* V, u64 n, u64 rl, const double* scales_dev, double* st, cudaStream_t s);
// For each candidate plane P: fixed-plane decoded stream -> reflectors ->
// Householder expansion; returns res[plane_idx * rl + j] =
// sum_i (X(i,j) - flip_j U(i,live_j))^2 (the host combines with the slice norms)
std::vector<double> factor_residuals(const u64* mag, const u8* neg, int k, u64 n, u64 r,
                                     const std::vector<u64>& live, const double* scales_dev, const double* U,
                                     const signed char* flips_dev, const std::vector<int>& planes, cudaStream_t s);
// Decoder: decoded reflector stream (mag, neg, k; column scales) -> U (row-major
// n x r; dead columns zero) by the Householder expansion (factor_codec.cpp:246-264)
void factor_expand(const u64* mag, const u8* neg, int k, u64 n, u64 r, const std::vector<u64>& live,
                   const double* scales_dev, double* U, cudaStream_t s,
                   int* err_dev = nullptr);

}  // namespace tcb
