// Ozaki-scheme digit products on the 5th-generation tensor cores (tcgen05,
// kind::i8): TMA-staged operands, int32 accumulators in tensor memory, the
// five digit levels combined exactly in int64 by the epilogue.  See ozmma.cu.
#pragma once

#include <vector>

#include "common.cuh"

namespace tcb {

constexpr int kOzSlices = 5;
constexpr u32 kOzBM = 128, kOzBN = 96;  // row blocks of the M (TMEM lane) and N operands
constexpr u64 kOzSlab = 64;             // bytes of k per slab

// Blocked digit layout: rows in blocks of br (kOzBM or kOzBN), k in 64-byte slabs;
// block blk, slab q holds the five slices back to back, each br rows of 64
// bytes, 16-byte chunks already in the 64-byte swizzle of the tensor core's
// shared-memory descriptor -- so one plain bulk copy per operand per slab
// fills a pipeline stage (TMA row-box loads of 64-byte rows ran at ~25 B/clk
// per SM, bulk copies of 30-40 KB at > 80, tools/dbg/tma_rate.cu).
__host__ __device__ inline u64 oz_block_off(u64 row, u64 k, int s, u32 br, u64 nslab) {
    const u64 blk = row / br, r = row % br, q = k / kOzSlab, kb = k % kOzSlab;
    return ((blk * nslab + q) * kOzSlices + static_cast<u64>(s)) * br * kOzSlab + r * kOzSlab +
           ((((kb >> 4) ^ (r >> 1)) & 3) << 4) + (kb & 15);
}
inline u64 oz_block_rows(u64 rows, u32 br) { return (rows + br - 1) / br * br; }
inline u64 oz_block_bytes(u64 rows, u64 nslab, u32 br) { return oz_block_rows(rows, br) * nslab * kOzSlices * kOzSlab; }

// Gram of a digit-sliced rows x (64 nslab) matrix given in both blockings
// (DA: 128-row blocks, DB: 96-row blocks): acc (int64, ld = acc_ld, rows padded
// to 128) += sum over levels L <= 4 of 2^(7 (4 - L)) sum_{s + t = L} d_s d_t^T,
// lower triangle incl. the diagonal valid; acc zeroed by the caller; nslab a
// multiple of 512 (2^15-byte k-chunks: int32-exact accumulation).
void oz_gram_tc(const int8_t* DA, const int8_t* DB, u64 rows, u64 nslab, long long* acc, u64 acc_ld, cudaStream_t s);
// the same for a subset of the (128-row a, 96-row b) tiles: the accumulation is
// exact integer, so any partition of the tiles over launches gives the same acc
void oz_gram_tc_tiles(const int8_t* DA, const int8_t* DB, u64 rows, u64 nslab, const std::vector<int2>& tiles,
                      long long* acc, u64 acc_ld, cudaStream_t s);
u64 oz_gram_acc_ld(u64 rows);  // the accumulator's leading dimension (tile-padded)

// TTM: A (m_rows, 128-row blocks), B (n_rows, 96-row blocks), nslab <= 64 ->
// out[c * n_rows + j] = sum_L 2^(7 (4 - L)) sum_{s + t = L} e_s . f_t * 2^(exa[c] + exb[j] - 40)
void oz_ttm_tc(const int8_t* A, u64 m_rows, const int8_t* B, u64 n_rows, u64 nslab, const int* exa, const int* exb,
               double* out, cudaStream_t s);

}  // namespace tcb
