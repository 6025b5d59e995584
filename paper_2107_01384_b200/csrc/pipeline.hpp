// Host orchestration of the device compress path (pipeline.cpp:24-195).
#pragma once

#include <array>
#include <exception>
#include <cmath>
#include <functional>
#include <optional>

#include "common.cuh"
#include "encoder.hpp"

namespace tcb {

struct Params {
    std::optional<double> target_re, target_sse;
    double rtmss = 0.5;
    int threads = 1;
    int method = 0;
    std::optional<std::vector<u64>> storage_order, mode_order;
    int coder = 0;
    bool split = true;
    bool simple = false;
    u64 block = 0;
    bool f32 = false;
    int backend = 0;
};

struct Times {
    double sthosvd = 0, quantize = 0, core = 0, factor = 0, serialize = 0, total = 0;
};

// Container bytes handed to the caller.  The memory comes from the result
// allocator (the C ABI installs its pinned-block pool, so the core payload's
// device-to-host copy lands in place at full PCIe rate); release() passes
// ownership on.
void set_result_allocator(void* (*alloc)(std::size_t), void (*release)(void*));
struct HostBytes {
    u8* p = nullptr;
    std::size_t n = 0;
    HostBytes() = default;
    explicit HostBytes(std::size_t bytes);
    HostBytes(const HostBytes&) = delete;
    HostBytes& operator=(const HostBytes&) = delete;
    HostBytes(HostBytes&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    HostBytes& operator=(HostBytes&& o) noexcept;
    ~HostBytes();
    u8* data() { return p; }
    const u8* data() const { return p; }
    std::size_t size() const { return n; }
    u8* release() {
        u8* q = p;
        p = nullptr;
        n = 0;
        return q;
    }
    static HostBytes from(const std::vector<u8>& v);
};

struct Result {
    HostBytes container;
    double trunc = 0, core_quant = 0, estimate = 0, norm_sq = 0, target_sse = 0;
    std::vector<double> factor_terms;
    std::vector<u64> ranks;
    Times times;
    u64 peak_alloc = 0, original_bytes = 0;
    bool precision_loss = false;
    int core_last_plane = 63, core_k = 0, uncertified = 0;
    unsigned rank_tie_modes = 0;
};

// device_bytes: element bytes (skip already applied) resident on the device
// gram0 (optional): the first mode's Gram of the fp64 input, already computed
// (bitwise as the mode loop would; the host entry point overlaps it with the upload)
// precast (optional, fp32 source): the input already cast to fp64 (moved from)
struct ShardComm;  // below
Result compress_device(const void* device_bytes, u64 nbytes, int dtype, const std::vector<u64>& shape,
                       const Params& p, cudaStream_t s,
                       const double* gram0 = nullptr,
                       const ShardComm* shard = nullptr,
                       DevBuf<double>* precast = nullptr);

struct Tucker {
    DevBuf<double> core;
    std::vector<u64> core_shape;
    std::vector<DevBuf<double>> factors;  // n_i x r_i row-major, by original mode
    std::vector<u64> n, r, order;
    std::vector<double> trunc;
    unsigned tie_modes = 0;  // bit i: mode i's rank decision sat in the tie band
};
// Sharded mode loop: the input is this rank's slab of the last
// processed mode (equal slabs, rank order); the Grams of steps 0..d-2 are
// summed over the ranks with NCCL before the eigensolve (so every rank holds
// the same factor), the TTMs stay shard-local, and the last step all-gathers
// the small projected tensor.  Steps 0..d-2 must take the Gram route.
// Collectives on host memory supplied by the caller (C ABI tcb_host_collectives):
// lets the sharded pipeline run over any transport (e.g. torch.distributed gloo)
struct HostCollectives {
    void* ctx;
    int (*allreduce_sum_f64)(void* ctx, double* buf, u64 n);                            // in place
    int (*allgather)(void* ctx, const void* send, void* recv, u64 bytes_per_rank);      // rank-major recv
};
struct ShardComm {
    void* comm = nullptr;                   // ncclComm_t (nccl_shim), or
    const HostCollectives* host = nullptr;  // host-memory collectives through caller callbacks
    int world = 1, rank = 0;
    u64 local_extent = 0;   // this rank's slab of mode p[d-1]
    // collectives on device buffers, ordered on s
    void allreduce_sum_f64(double* d, u64 n, cudaStream_t s) const;
    void allgather(const void* dsend, void* drecv, u64 bytes_per_rank, cudaStream_t s) const;
    // host blobs of any size, one per rank
    std::vector<std::vector<u8>> allgather_blobs(const std::vector<u8>& mine, cudaStream_t s) const;
};

// One mode step (sthosvd.cpp:136-166): factor U (rows x r, sign-fixed), the
// discarded energy, and the projected/shifted tensor next = B^T U (cols x r).
struct StepOut {
    u64 r = 0;
    double discarded = 0.0;
    bool tie = false;  // the budget lies within the eigenvalues' error band of a cutoff
    DevBuf<double> U, next;
};
// A mode step's SSE budget: a fixed value, or `scale` x trace(G) of the step's
// Gram -- on the first step trace(B B^T) = |A|_F^2, so the input norm comes with
// the Gram instead of a separate pass.  The trace used is reported.
struct TraceNonFinite {};  // the Gram's trace is not finite (scan the input)
struct Budget {
    double value = 0.0;
    double scale = -1.0;
    double* trace_out = nullptr;
    Budget(double v = 0.0) : value(v) {}  // NOLINT: implicit from a fixed budget
    double eval(double trace) const {
        if (trace_out) {
            *trace_out = trace;
            if (!std::isfinite(trace)) throw TraceNonFinite{};
        }
        return scale < 0 ? value : scale * trace;
    }
};
// gram (optional): this step's Gram B B^T already computed (rows <= cols branch)
StepOut mode_step(const double* x, u64 rows, u64 cols, const Budget& budget, int backend, cudaStream_t s,
                  const double* gram = nullptr, const ShardComm* shard = nullptr);
// eigensolve + rank rule + sign fix on an (all-reduced) Gram; U is n x r
StepOut factor_from_gram(const double* G, u64 n, const Budget& budget, cudaStream_t s, bool tail_from_trace = false);
// sthosvd::compress (sthosvd.cpp:114-171) on a device tensor.  The input is
// `ext` when non-null (read-only, e.g. the caller's fp64 buffer: with an
// identity processing order mode 0 reads it in place), else `owned`, which is
// released as soon as it is no longer needed.  finite: 1 / 0 when the caller
// already scanned the values (the norm pass), -1 to scan here.
// on_factor (optional) is called after each mode step with (mode, U, n, r), U
// complete on `s`.
// norm_scale >= 0: the target is norm_scale x |A|_F^2 with the norm read off the
// first Gram's trace (written to *norm_out; TraceNonFinite when it is not finite).
Tucker sthosvd_device(DevBuf<double>&& owned, const double* ext, const std::vector<u64>& shape, double target,
                      const std::optional<std::vector<u64>>& order, int backend, cudaStream_t s, int finite = -1,
                      const std::function<void(std::size_t, const double*, u64, u64)>& on_factor = {},
                      double norm_scale = -1.0, double* norm_out = nullptr, const double* gram0 = nullptr,
                      const ShardComm* shard = nullptr);
inline Tucker sthosvd_device(DevBuf<double>&& a, const std::vector<u64>& shape, double target,
                             const std::optional<std::vector<u64>>& order, int backend, cudaStream_t s) {
    return sthosvd_device(std::move(a), nullptr, shape, target, order, backend, s);
}

struct FactorEnc {
    std::vector<u8> dead;
    std::vector<double> slice_norms;
    int k = 0;
    u64 count = 0;
    std::vector<u8> stream;  // serialized section
    std::vector<signed char> flips;
    double term = 0;
    int plane = 0;
};
// Phases 2-5 of compress_impl on an existing device factorization (used by
// the sharded multi-GPU mode loop, whose rank 0 encodes the gathered core).
Result encode_tucker_device(Tucker& f, int dtype, double norm_sq, double target, const Params& p, cudaStream_t s,
                            const ShardComm* shard = nullptr);

// The orthonormality check and Householder reflectors of a factor's live
// columns (factor_codec.cpp:29-31,153-200); an error is captured in `err` and
// rethrown when the factor is actually encoded.
struct FactorPrep {
    std::vector<u64> live;
    DevBuf<double> V;               // n x live reflectors
    std::vector<signed char> fl;    // per live column
    std::exception_ptr err;
};
FactorPrep factor_prepare(const double* U, u64 n, u64 r, const std::vector<u8>& dead, bool f32, cudaStream_t s);
// The quantised reflector stream of a factor for a given live set
// (factor_codec.cpp:200-217) and, once the core's last plane is known, the
// plane search over it (factor_codec.cpp:218-243): computed speculatively for
// "no dead columns" while the core plan runs, reused when the plan agrees.
struct FactorQuant {
    std::vector<u64> live;
    std::vector<double> ln, sc;
    DevBuf<double> dsc;
    DevBuf<signed char> dfl;
    u64 cnt = 0;
    int k = 0;
    DevBuf<u64> mag;
    DevBuf<u8> neg;
    int core_step = 1 << 30;  // the core step the plane search below was made for
    int plane = -1;
    double term = 0.0;
    std::vector<u8> stream;   // the finalised stream section for `plane` (when `finalized`)
    bool finalized = false;
};
// finalise q's stream section for its plane (factor_codec.cpp:244, core_codec.cpp:328-391)
void factor_finalize(FactorQuant& q, int coder, cudaStream_t s);
void factor_quantize(FactorQuant& q, const FactorPrep& prep, u64 n, const std::vector<double>& sn_live, bool simple,
                     cudaStream_t s);
void factor_plane_search(FactorQuant& q, const double* U, u64 n, u64 r, int core_step_log2, double cap,
                         cudaStream_t s);
// on_flips (optional) receives the column sign flips as soon as they are known,
// before the plane search and stream finalisation; `prep` (optional) is reused
// when it was made for the same live columns.
FactorEnc encode_factor_device(const double* U, u64 n, u64 r, const std::vector<u8>& dead,
                               const std::vector<double>& sn, int coder, bool simple, int core_step_log2,
                               double cap, bool f32, cudaStream_t s,
                               const std::function<void(const std::vector<signed char>&)>& on_flips = {},
                               FactorPrep* prep = nullptr, FactorQuant* spec = nullptr);

std::vector<double> alpha_weights(const std::vector<double>& sn, u64 n);
std::vector<u64> stable_ascending(const std::vector<u64>& s);

}  // namespace tcb
