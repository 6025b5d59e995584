// Exact parallel evaluation of the reference encoder's SERIAL double sums.
//
// The reference decides its breakpoint plane, recalibrations and stop
// positions by comparing doubles it accumulates one term at a time
// (error_model.cpp:34-72, core_codec.cpp:137-153,183,268-341,405-411).  This
// engine returns, bit for bit, the double `s` that loop ends with
//     s = s0; for i in order: s = fl(s + t_i)
// without running the dependent chain element by element:
//
// * every term t_i is an integer-valued double, so while the running sum
//   stays inside one binade region R (|s| in [2^e, 2^(e+1)), or |s| < 2^53)
//   every s is an integer multiple a*u of u = 2^(e-52) and
//       fl(s + t) = (a + round_half_even(a + t/u) - a) u,
//   which advances a by round(t/u) independently of a -- except at exact
//   ties, where the result is the even neighbour: a two-state transducer in
//   the parity of a.  A run of terms is therefore summarised, for a given R,
//   by a function of the start parity: (increment K, end parity, min/max
//   partial increment) per parity.  These compose associatively.
// * pass 1 sums each chunk approximately, a scan turns those into each
//   chunk's approximate starting value, whose region is the guess R_c;
//   pass 2 builds every chunk's function for R_c;
// * a walk (one warp per sum) applies 32 chunk functions per step (warp
//   scan of the compositions) and accepts a chunk only when its start value
//   is really in R_c and every partial sum stays strictly inside R_c (so the
//   rounding unit was u throughout); a rejected chunk -- a region change or a
//   wrong guess, a few per binade crossing -- is re-resolved by the warp
//   with 8-term functions built for the actual region and a plain serial
//   __dadd_rn chain only across the lane where the region changes.
//
// Crossing scans (place_stops) run the same walk with a threshold `need`:
// the first element after which s >= need, found exactly.
#pragma once

#include <cmath>
#include <memory>
#include <vector>

#include "common.cuh"

namespace tcb {

enum ExTerm : int {
    kExLead = 0,   // plane p: msb == p -> lead gain; category positions msb <= p
    kExTrail = 1,  // plane p: msb > p -> trail gain; category positions msb > p
    kExBoth = 2,   // plane p: both (the non-split interleaved scan)
    kExSq = 3,     // (double)m squared (backward_sum_sse)
    kExRecal = 4,  // recalibrate_sse term at plane p
    kExDiff = 5,   // ((double)m - (double)dec)^2 (achieved SSE)
};

struct ExKind {
    int term;
    int plane;
};

// A serially summed run of elements: indices [lo, hi) in ascending order, or
// descending when `backward`; the sum starts from s0.  need < +inf makes it a
// crossing scan (stop after the first element that brings s to >= need).
struct ExSeg {
    u64 lo, hi;
    int backward;
    double s0;
    double need;
};

struct ExOut {
    double sum;   // the serial sum (at the crossing element when crossed)
    u64 c0, c1;   // category counts: lead positions / trail positions (lead: c1 = new ones); up to the crossing
    int crossed;
};

// Every (kind, segment) pair: out[k * segs.size() + g].  `dec` is read only by kExDiff.
// TCB_EXACT_REFERENCE=1 routes every call through exact_serial_reference.
std::vector<ExOut> exact_serial(const u64* m, const u64* dec, const std::vector<ExSeg>& segs,
                                const std::vector<ExKind>& kinds, cudaStream_t s);

// build_block's per-block statistics of planes p_top .. p_top - np + 1 (np <= 32)
// over blocks of `block` elements: out[k * nb + b] with kinds k = 2 (p_top - p)
// + {0: lead, 1: trail}, as exact_serial would return them.
std::vector<ExOut> exact_plane_stats(const u64* m, u64 n, u64 block, int p_top, int np, cudaStream_t s);

// The same in two steps: approx_residuals() estimates, from a 1/64 sample of
// the elements, the squared error left after coding each plane p_top ..
// p_top - np + 1 in full (sum over msb >= p of sig(m, p), over msb < p of m^2:
// a sum of non-negative terms, so a sample estimates it to a relative error,
// unlike the difference `tracked - sum of reductions`), so the caller can
// estimate how many planes it needs; exact(np_exact) returns the exact
// statistics of the first np_exact planes only (elements below them skipped).
class PlaneStatsJob {
public:
    // blocks [b0, b1) only (a rank's share); results index k * (b1 - b0) + (b - b0)
    PlaneStatsJob(const u64* m, u64 n, u64 block, int p_top, int np, cudaStream_t s, u64 b0 = 0,
                  u64 b1 = ~u64{0});
    ~PlaneStatsJob();
    std::vector<double> approx_residuals();
    std::vector<ExOut> exact(int np_exact);

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
    cudaStream_t s_;
};

// Debug/verification: the same sums by the plain one-thread serial chain.
std::vector<ExOut> exact_serial_reference(const u64* m, const u64* dec, const std::vector<ExSeg>& segs,
                                          const std::vector<ExKind>& kinds, cudaStream_t s);

// one backward sum over a whole array (backward_sum_sse, recalibrate_sse, achieved SSE)
inline double exact_backward_sum(int term, int plane, const u64* m, const u64* dec, u64 n, cudaStream_t s) {
    if (n == 0) return 0.0;
    return exact_serial(m, dec, {ExSeg{0, n, 1, 0.0, HUGE_VAL}}, {ExKind{term, plane}}, s)[0].sum;
}

}  // namespace tcb
