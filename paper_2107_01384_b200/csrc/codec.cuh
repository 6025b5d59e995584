// Bit-plane codec kernels (core_codec.cpp / entropy.cpp / error_model.cpp).
#pragma once

#include <functional>

#include <memory>
#include <utility>
#include <vector>

#include "common.cuh"

namespace tcb {

// Exact-sum record for one serially accumulated double sum the reference
// makes: hi+lo is the (double-double) exact value of the term sum, `wabs` a
// bound on sum_k |partial_k| used to bound the serial rounding error.
struct SumRec {
    double hi, lo, wabs;
    u64 nterms;
};

// Per (plane, block) statistics of build_block (core_codec.cpp:120-171).
struct PlaneBlockRec {
    SumRec lead, trail;
    u64 nlead, nones, ntrail;
};

enum class SumKind : int { sq_backward = 0, recal_backward = 1, diff_backward = 2 };

// sum over i of term_i (error_model.cpp:34-72, core_codec.cpp:405-411)
SumRec device_sum(SumKind kind, const u64* m, const u64* dec, u64 n, int plane, cudaStream_t s);
// exact serial replay (fallback when a decision cannot be certified)
double device_sum_serial(SumKind kind, const u64* m, const u64* dec, u64 n, int plane, cudaStream_t s);

// stats for planes [p_lo, p_hi], out[(p_hi - p) * nb + b]
void plane_stats(const u64* m, u64 n, u64 block, int p_hi, int p_lo, PlaneBlockRec* out_host, cudaStream_t s);
// exact serial replay of the per-block sums for one plane
void plane_stats_serial(const u64* m, u64 n, u64 block, int p, PlaneBlockRec* out_host, cudaStream_t s);
// the exact statistics of planes p_hi..p_lo at once (plane-major: (p_hi - p) * nb + block)
void plane_stats_serial_range(const u64* m, u64 n, u64 block, int p_hi, int p_lo, PlaneBlockRec* out_host,
                              cudaStream_t s);
// several serial sums (kind, plane) over m at once, each in its own CTA
std::vector<double> device_sums_serial(const std::vector<std::pair<SumKind, int>>& list, const u64* m, u64 n,
                                       cudaStream_t s);

// Crossing scan of place_stops (core_codec.cpp:268-341): count positions of the
// given category in block b until cum >= need; returns counts for (cum, need).
// category: 0 = leading, 1 = trailing, 2 = interleaved (non-split).
void crossing_scan(const u64* m, u64 n, u64 block, u64 b, int plane, int category, const double* cum,
                   const double* need, int npairs, u64* counts_host, cudaStream_t s);

// per-block histogram of the magnitudes' top bit: nb x 65 (bins <-> msb -1..63)
std::vector<u64> msb_histogram(const u64* m, u64 n, u64 block, cudaStream_t s);

// decoded magnitudes implied by (last_plane, stops) (core_codec.cpp:344-367)
void decode_model(const u64* m, u64 n, u64 block, int last_plane, const u64* stops_dev /*2*nb*/, u64* dec,
                  cudaStream_t s);

// One encoded stream: planes [last_plane .. 63] x blocks; returns the section
// bytes "nplanes-major (u32 size || payload)" exactly as write_stream lays out
// the payload part (container.cpp:240-246).
struct EmitResult {
    std::vector<u8> body;  // concatenated (u32 size || payload) for every (plane, block)
    std::vector<u64> entropy_bytes;  // per stream, for split-plane priority probes
};
// A contiguous range of blocks [b0, b1) (a rank's share under sharded
// encoding); the default is every block.
struct BlockRange {
    u64 b0 = 0, b1 = ~u64{0};
};
// the same with the assembled body left in device memory; streams are plane-major
// over the range's blocks, stream_bytes[i] = 4 + payload of stream i
struct EmitDev {
    DevBuf<u8> body;
    u64 size = 0;
    std::vector<u64> entropy_bytes;
    std::vector<u64> stream_bytes;
};
// `hist` (optional): the per-block msb histogram (msb_histogram) when the caller has it
EmitDev emit_planes_device(const u64* m, const u8* neg, u64 n, u64 block, int last_plane, int top_plane,
                           const u64* stops_host, int coder, cudaStream_t s, BlockRange br = {},
                           const std::vector<u64>* hist = nullptr);
EmitResult emit_planes(const u64* m, const u8* neg, u64 n, u64 block, int last_plane, int top_plane,
                       const u64* stops_host /*2*nb, for last_plane*/, int coder, bool want_body,
                       cudaStream_t s, BlockRange br = {});

// Arithmetic-coder size bounds [lo, hi] of plane `plane`'s full streams (blocks of
// the range; out[2 i], out[2 i + 1]) from the adaptive model alone: enough to
// decide the split-plane priority without the sequential range pass, usually.
// `launched` (optional) runs once every kernel is enqueued, before the host waits.
std::vector<u64> entropy_size_bounds(const u64* m, u64 n, u64 block, int plane, cudaStream_t s, BlockRange br = {},
                                     const std::function<void()>& launched = {});

// Speculative split-plane probe: the entropy-coded size of every full plane
// stream (planes 63..0, no stops, signs not needed) launched on a side stream
// as soon as the magnitudes exist, so the planner's probe of plane p+1
// (core_codec.cpp:244-290) is a lookup instead of a round trip on the
// critical path.
struct ProbeCache;
std::shared_ptr<ProbeCache> probe_planes_async(const u64* m, u64 n, u64 block, int coder, cudaStream_t side);
// entropy bytes of plane p's streams (one per block); waits for the side stream
std::vector<u64> probe_entropy_bytes(ProbeCache& c, int p);

// entropy::encode_symbols for one host symbol sequence (arithmetic coder)
std::vector<u8> encode_symbols_device(int coder, const u64* syms_host, u64 n, cudaStream_t s);

}  // namespace tcb
