// Ozaki-scheme digit products on the 5th-generation tensor cores (tcgen05,
// kind::i8): TMA-staged operands, int32 accumulators in tensor memory, the
// five digit levels combined exactly in int64 by the epilogue.  See ozmma.cu.
#pragma once

#include "common.cuh"

namespace tcb {

constexpr int kOzSlices = 5;

// Gram of a digit-sliced rows x K matrix: D (rows_p x 5 Kp bytes, row i =
// [d_0 | .. | d_4], each Kp long, zero padded) -> acc (int64, rows x rows,
// lower triangle incl. the diagonal valid, ld = acc_ld) += sum over levels
// L <= 4 of 2^(7 (4 - L)) sum_{s + t = L} d_s d_t^T (exact integers).
// `acc` must be zeroed by the caller; Kp a multiple of 2^15.
void oz_gram_tc(const int8_t* D, u64 rows, u64 rows_p, u64 Kp, long long* acc, u64 acc_ld, cudaStream_t s);
u64 oz_gram_acc_ld(u64 rows);  // the accumulator's leading dimension (tile-padded)

// TTM: A (m_rows x 5 Ka bytes, row c = [e_0 | .. | e_4]), B (n_rows x 5 Ka) ->
// out[c * n_rows + j] = scalbn(sum_L 2^(7 (4 - L)) sum_{s + t = L} e_s . f_t, exa[c] + exb[j] - 40)
// for c < m_rows, j < n_rows; Ka a multiple of 64, at most 4096.
void oz_ttm_tc(const int8_t* A, u64 m_rows, const int8_t* B, u64 n_rows, u64 Ka, const int* exa, const int* exb,
               double* out, cudaStream_t s);

}  // namespace tcb
