// Adaptive range coder of the bit-plane streams (entropy.cpp:85-239) on the
// device, bit-exact, as three passes over every stream at once:
//
// 1. model: one CTA per stream resolves the adaptive model
//    (AdaptiveModel::encode / bump / insert / halve) 256 symbols at a time --
//    between halvings every count is its value at the chunk start plus 32 per
//    earlier occurrence, so (cum, freq, total) of each symbol is a dominance
//    count inside the chunk plus a prefix of the chunk-start counts;
// 2. range: one warp per stream runs the only truly sequential part, the
//    32-bit range recurrence  range = norm(floor(range / total) * freq)
//    (division by a per-symbol multiply-high), and records W[S] = the sum of
//    the cum * (range / total) additions made while S bytes had been shifted
//    out -- the carry-propagating `low` register is never materialised;
// 3. bytes: the output is the big-endian digit string of
//    Z = sum_S W[S] * 256^(N-5-S)  (N = number of shift_low calls), so each
//    byte is a 5-term digit sum plus a carry resolved by a parallel
//    generate/propagate scan.
#pragma once

#include <functional>
#include <vector>

#include "common.cuh"

namespace tcb {

struct AcJob {
    u64 sym_off;    // first symbol of the stream in `syms`
    u64 out_off;    // output position in `ent` (capacity ac_out_cap)
    u64 sym_cap;    // symbol-count bound (the actual count is read on the device)
    u64 positions;  // column length (bounds the number of distinct run lengths)
    u64 distinct = 0;  // a tighter bound on the distinct symbols when known (0: from positions)
};

// distinct run lengths of a column with `positions` bits: d(d-1)/2 <= zeros
u64 ac_escape_bound(u64 sym_cap, u64 positions);
// bytes of encode_symbols output (u8 coder || u32 count || range-coder body)
u64 ac_out_cap(u64 sym_cap, u64 positions);

// Codes every stream: symbols syms[job.sym_off + i], i < counts[j * stride]
// (device), into ent + job.out_off; elen[j] = total bytes, 0 for no symbols.
// err_dev (zeroed by the caller): no host sync here -- the flag is set on a
// model-capacity overflow and the caller checks it with its results; null:
// checked (synchronously) before returning.
void ac_encode(const u64* syms, const u64* counts, int stride, const std::vector<AcJob>& jobs, u8* ent, u64* elen,
               cudaStream_t s, int* err_dev = nullptr);

// Bounds [lo, hi] (out[2 j], out[2 j + 1]) on each stream's encode_symbols size from
// the adaptive model alone (no range recurrence); lo == hi == 0 for no symbols.
// `launched` (optional) runs once every kernel is enqueued, before the wait.
std::vector<u64> ac_size_bounds(const u64* syms, const u64* counts, int stride, const std::vector<AcJob>& jobs,
                                cudaStream_t s, const std::function<void()>& launched = {});

}  // namespace tcb
