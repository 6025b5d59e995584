// Host orchestration of the B200 compress path, mirroring compress_impl
// (pipeline.cpp:24-195), sthosvd::compress (sthosvd.cpp:114-171) and
// factorcodec::encode_factor (factor_codec.cpp:153-244).  All tensor work runs
// in the device kernels; the host keeps the reference's scalar decisions
// (rank rule, budget roll-forward, plane deepening) in the same double
// arithmetic (no FMA contraction in this TU).
#include "pipeline.hpp"

#include <algorithm>
#include <atomic>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <future>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <thread>
#include <tuple>

#include "exact.cuh"
#include "kernels.cuh"
#include "nccl_shim.hpp"
#include "quant.cuh"

namespace tcb {

namespace {
// Host worker pool for the concurrent factor encodes: persistent threads (a
// thread per call would cost more than the overlap saves) and one
// non-blocking CUDA stream per (device, slot).
class Workers {
public:
    static Workers& get() {
        static Workers w;
        return w;
    }
    std::future<void> submit(std::function<void()> f) {
        auto task = std::make_shared<std::packaged_task<void()>>(std::move(f));
        auto fut = task->get_future();
        {
            std::lock_guard<std::mutex> lk(m_);
            q_.push_back([task] { (*task)(); });
        }
        cv_.notify_one();
        return fut;
    }
    cudaStream_t stream(int dev, int slot) {
        std::lock_guard<std::mutex> lk(m_);
        auto& v = streams_[dev];
        while (static_cast<int>(v.size()) <= slot) {
            cudaStream_t st;
            TCB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            v.push_back(st);
        }
        return v[slot];
    }

private:
    Workers() {
        for (int i = 0; i < 8; ++i) th_.emplace_back([this] { run(); });
    }
    ~Workers() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void run() {
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
                if (stop_ && q_.empty()) return;
                f = std::move(q_.front());
                q_.pop_front();
            }
            f();
        }
    }
    std::mutex m_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    std::vector<std::thread> th_;
    std::map<int, std::vector<cudaStream_t>> streams_;
    bool stop_ = false;
};
// waits for every submitted task before the stack data they reference unwinds
struct JoinAll {
    std::vector<std::future<void>>& f;
    ~JoinAll() {
        for (auto& x : f)
            if (x.valid()) x.wait();
    }
};
}  // namespace


namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) { return std::chrono::duration<double, std::milli>(Clock::now() - t0).count(); }

bool valid_perm(const std::vector<u64>& p, std::size_t d) {
    if (p.size() != d) return false;
    std::vector<char> seen(d, 0);
    for (auto v : p) {
        if (v >= d || seen[v]) return false;
        seen[v] = 1;
    }
    return true;
}

std::size_t dtype_size(int t) {
    switch (t) {
        case 0: case 1: return 1;
        case 2: case 3: return 2;
        case 4: case 5: case 8: return 4;
        case 6: case 7: case 9: return 8;
    }
    throw Error("container: unknown dtype");
}

// SURVEY H3 tie band: the rank rule compares tail sums of eigenvalues with the
// budget; a solver's eigenvalues carry an absolute error of a few n eps |G|, so
// when the budget is closer than that to the sum at the chosen cutoff or at the
// next one, another correct fp64 solver (the reference's) may cut one vector
// earlier or later.  Reported, not corrected.
bool rank_tie(const std::vector<double>& s2, u64 r, double gone, double budget) {
    if (s2.empty()) return false;
    const double n = static_cast<double>(s2.size());
    const double err = 8.0 * n * DBL_EPSILON * std::max(s2[0], 0.0) * std::sqrt(n - static_cast<double>(r) + 1.0);
    const double keep_next = r > 0 ? gone + s2[r - 1] : gone;  // the sum that stopped the discard loop
    return std::fabs(budget - gone) <= err || std::fabs(keep_next - budget) <= err;
}

// sthosvd.cpp:13-26
std::pair<u64, double> pick_rank(const std::vector<double>& s2, double budget) {
    if (s2.empty()) throw Error("rank choice: empty singular values");
    if (budget < 0) throw Error("rank choice: negative budget");
    u64 r = s2.size();
    double gone = 0.0;
    while (r > 0) {
        const double next = gone + s2[r - 1];
        if (next > budget) break;
        gone = next;
        --r;
    }
    return {r, gone};
}

struct W {
    std::vector<u8> b;
    void u8v(u8 v) { b.push_back(v); }
    void u32v(u32 v) {
        for (int i = 0; i < 4; ++i) b.push_back(static_cast<u8>(v >> (8 * i)));
    }
    void u64v(u64 v) {
        for (int i = 0; i < 8; ++i) b.push_back(static_cast<u8>(v >> (8 * i)));
    }
    void f64v(double v) {
        u64 x;
        std::memcpy(&x, &v, 8);
        u64v(x);
    }
    void raw(const std::vector<u8>& x) { b.insert(b.end(), x.begin(), x.end()); }
};

std::vector<u8> empty_stream_section(u64 count, u64 block) {
    W w;
    w.u64v(count);
    w.u64v(block);
    w.u8v(63);
    w.u32v(0);
    w.u32v(0);
    return w.b;
}

__attribute__((unused)) void sync(cudaStream_t s) { stream_sync(s); }

}  // namespace

namespace {
void* (*g_res_alloc)(std::size_t) = nullptr;
void (*g_res_release)(void*) = nullptr;
}  // namespace

void set_result_allocator(void* (*alloc)(std::size_t), void (*release)(void*)) {
    g_res_alloc = alloc;
    g_res_release = release;
}

HostBytes::HostBytes(std::size_t bytes) : n(bytes) {
    p = static_cast<u8*>(g_res_alloc ? g_res_alloc(bytes + 1) : std::malloc(bytes + 1));
    if (!p) throw Error("compress: out of host memory");
}
HostBytes& HostBytes::operator=(HostBytes&& o) noexcept {
    if (this != &o) {
        this->~HostBytes();
        p = o.p;
        n = o.n;
        o.p = nullptr;
        o.n = 0;
    }
    return *this;
}
HostBytes::~HostBytes() {
    if (p) (g_res_release ? g_res_release : std::free)(p);
    p = nullptr;
}
HostBytes HostBytes::from(const std::vector<u8>& v) {
    HostBytes h(v.size());
    if (!v.empty()) std::memcpy(h.p, v.data(), v.size());
    return h;
}

std::vector<u64> stable_ascending(const std::vector<u64>& s) {
    std::vector<u64> p(s.size());
    std::iota(p.begin(), p.end(), u64{0});
    std::stable_sort(p.begin(), p.end(), [&](u64 a, u64 b) { return s[a] < s[b]; });
    return p;
}

std::vector<double> alpha_weights(const std::vector<double>& sn, u64 n) {
    const std::size_t r = sn.size();
    if (n < r) throw Error("weights: factor has more columns than rows");
    std::vector<double> al(r);
    double tail = 0.0;
    for (std::size_t k = 0; k < r; ++k) tail += sn[k] * sn[k];
    for (std::size_t j = 0; j < r; ++j) {
        const double sj = sn[j];
        tail -= sj * sj;
        const double nj = static_cast<double>(n - j);
        const double q = std::sqrt(nj);
        const double own = 1.0 + (nj + 5.0 * q + 2.0) / ((q + 1.0) * (q + 1.0) * q);
        al[j] = own * sj * sj;
        if (tail > 0.0) {
            const double tc = 2.0 / (nj - 1.0) + (nj + 2.0 * q + 2.0) / ((q + 1.0) * (q + 1.0) * (q + 1.0) * q);
            al[j] += tc * tail;
        }
    }
    return al;
}

// Fast path of the eigensolve + rank rule (topk.cu): top-32 Ritz pairs by
// block subspace iteration, accepted only with a certificate --
//   * the rank rule's cutoff r leaves >= 8 vectors of the block unused, with
//     the discarded energy taken as trace(G) - sum_{j<r} theta_j;
//   * every kept residual |G x_j - theta_j x_j| is at the roundoff floor
//     (16 eps sqrt(n) theta_0), so |theta_j - lambda_j| is negligible;
//   * the Davis-Kahan bound |R_kept|_F / (theta_{r-1} - theta_r - |r_r|) on
//     the kept subspace's sine is <= 5e-7 (the parity tolerance is 1e-6).
// V receives the n x r Ritz vectors (unsigned).  false: use the full solver.
bool topk_factor(const double* G, u64 n, const Budget& bud, cudaStream_t s, u64& r_out, double& gone_out,
                 std::vector<double>& s2_out, DevBuf<double>& V, bool* tie_out = nullptr) {
    constexpr int p = 32, spare = 8;
    if (!topk_supported(n, p)) return false;
    if (const char* e = std::getenv("TCB_NO_TOPK"); e && *e && *e != '0') return false;
    DevBuf<double> X(n * p, s);
    static const std::vector<int> attempts = [] {  // TCB_TOPK_ITERS="2,5": extra iterations per attempt
        std::vector<int> v;
        if (const char* e = std::getenv("TCB_TOPK_ITERS"); e && *e) {
            for (const char* c = e; *c;) {
                v.push_back(std::atoi(c));
                while (*c && *c != ',') ++c;
                if (*c) ++c;
            }
        }
        if (v.empty()) v = {2, 5};
        return v;
    }();
    for (int extra : attempts) {
        HostTrace ht(extra <= 1 ? "topk: attempt (extra<=1)" : extra <= 3 ? "topk: attempt (extra 2-3)" : "topk: attempt (extra>3)");
        std::vector<double> th, res;
        double tr = 0.0;
        topk_eig(G, n, p, extra, X.p, th, res, tr, s);
        const double budget = bud.eval(tr);
        std::vector<double> s2(p);
        for (int j = 0; j < p; ++j) s2[j] = std::max(0.0, th[j]);
        int r = -1;
        double gone = 0.0, pref = 0.0;
        for (int k = 0; k <= p - spare; ++k) {
            const double tail = std::max(0.0, tr - pref);
            if (tail <= budget) {
                r = k;
                gone = tail;
                break;
            }
            pref += s2[k];
        }
        if (r < 0) return false;  // cutoff beyond the block
        if (r == 0) {             // sthosvd.cpp:146-150
            r = 1;
            gone -= s2[0];
        }
        const double floor_res = 16.0 * DBL_EPSILON * std::sqrt(static_cast<double>(n)) * std::max(th[0], 0.0);
        double rk2 = 0.0, rmax = 0.0;
        for (int j = 0; j < r; ++j) {
            rk2 += res[j] * res[j];
            rmax = std::max(rmax, res[j]);
        }
        const double gap = th[r - 1] - th[r] - res[r];
        const bool ok = rmax <= floor_res && gap > 0.0 && std::sqrt(rk2) <= 5e-7 * gap;
        if (!ok) continue;
        r_out = static_cast<u64>(r);
        gone_out = gone;
        s2_out = s2;
        if (tie_out) {  // the tail beyond the block is trace - prefix: one more candidate sum
            const double err = 8.0 * static_cast<double>(n) * DBL_EPSILON * std::max(th[0], 0.0) *
                               std::sqrt(static_cast<double>(n) - r + 1.0);
            const double next = gone + s2[r - 1];
            *tie_out = std::fabs(budget - gone) <= err || std::fabs(next - budget) <= err;
        }
        V = DevBuf<double>(n * r, s);
        TCB_CUDA(cudaMemcpy2DAsync(V.p, r * sizeof(double), X.p, p * sizeof(double), r * sizeof(double), n,
                                   cudaMemcpyDeviceToDevice, s));
        return true;
    }
    return false;
}

// The discarded energy as trace(G) - (kept eigenvalues) instead of the sum of the
// clipped tail: for a Gram whose null space carries rounding noise of one sign
// more than the other (the INT8 path's truncated digit products), summing
// max(0, noise) over hundreds of null eigenvalues biases the tail upwards.
std::pair<u64, double> pick_rank_trace(const std::vector<double>& s2, double trace, double budget) {
    if (s2.empty()) throw Error("rank choice: empty singular values");
    if (budget < 0) throw Error("rank choice: negative budget");
    u64 r = 0;
    double kept = 0.0;
    while (r < s2.size() && std::max(0.0, trace - kept) > budget) kept += s2[r++];
    return {r, std::max(0.0, trace - kept)};
}

StepOut factor_from_gram(const double* G, u64 n, const Budget& bud, cudaStream_t s, bool tail_from_trace) {
    {
        StepOut o;
        std::vector<double> s2;
        if (topk_factor(G, n, bud, s, o.r, o.discarded, s2, o.U, &o.tie)) {
            fix_column_signs(o.U.p, n, o.r, s);
            return o;
        }
    }
    const double budget = bud.eval(bud.trace_out ? gram_trace(G, n, s) : 0.0);  // (checks the trace first)
    EigWork w;
    const auto ev = eig_values(G, n, w, s);
    std::vector<double> s2(n);
    for (u64 j = 0; j < n; ++j) s2[j] = std::max(0.0, ev[j]);
    auto [r, gone] = tail_from_trace ? pick_rank_trace(s2, gram_trace(G, n, s), budget) : pick_rank(s2, budget);
    const bool tie = rank_tie(s2, r, gone, budget);
    if (r == 0) {  // a budget above the whole mode energy still keeps one vector (sthosvd.cpp:146-150)
        r = 1;
        gone -= s2[0];
    }
    StepOut o;
    o.tie = tie;
    o.r = r;
    o.discarded = gone;
    o.U = DevBuf<double>(n * r, s);
    eig_vectors(w, r, o.U.p, s);
    fix_column_signs(o.U.p, n, r, s);
    return o;
}

StepOut mode_step(const double* x, u64 rows, u64 cols, const Budget& budget, int backend, cudaStream_t s,
                  const double* gram, const ShardComm* shard) {
    const bool sharded = shard && shard->world > 1;
    // rows > cols is the reference's thin-SVD branch (sthosvd.cpp:75-76,91-99): only
    // cols singular values exist, so r <= cols whatever the budget; the stand-in is
    // the Gram of B^T, U = B V / sigma, re-orthonormalised.  rows <= cols: the Gram
    // of B (for SvdBackend::direct too -- its thin U has the same rows columns).
    const u64 cols_all = sharded ? cols * static_cast<u64>(shard->world) : cols;
    const bool via_gram = backend == 1 || rows <= cols_all;
    if (sharded && !via_gram) throw Error("sharded compress: a step off the Gram route (rows > cols)");
    StepOut o;
    std::unique_ptr<OzTtmPrep> tprep;
    if (via_gram) {
        DevBuf<double> G;
        // a Gram handed in (the host upload's) is the one this step would compute:
        // the Ozaki one exactly where ozaki_gram_ok holds
        bool oz = gram && ozaki_gram_ok(rows, cols);
        if (!gram) {
            G = DevBuf<double>(rows * rows, s);
            if (ozaki_gram_ok(rows, cols)) {
                gram_ozaki(x, rows, cols, G.p, s);
                oz = true;
            } else {
                gram_f64(x, rows, cols, G.p, s);
            }
        }
        // the TTM's B-side digits need only x: on a low-priority side stream they
        // fill the eigensolve's latency-bound SMs (wasted when r < 64 or thin)
        if (ozaki_gram_ok(rows, cols) && rows <= 4096) {
            static PerDevice<cudaStream_t> prep_streams;
            cudaStream_t side = prep_streams.get([] {
                int lo = 0, hi = 0;
                TCB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
                cudaStream_t x2;
                TCB_CUDA(cudaStreamCreateWithPriority(&x2, cudaStreamNonBlocking, lo));
                return x2;
            });
            EventHandle q;
            TCB_CUDA(cudaEventRecord(q.e, s));
            TCB_CUDA(cudaStreamWaitEvent(side, q.e, 0));
            tprep = ttm_ozaki_prepare(x, rows, cols, side);
        }
        if (sharded) {  // the columns are spread over the ranks: sum the partial Grams
            if (gram) {
                G = DevBuf<double>(rows * rows, s);
                TCB_CUDA(cudaMemcpyAsync(G.p, gram, rows * rows * sizeof(double), cudaMemcpyDeviceToDevice, s));
            }
            shard->allreduce_sum_f64(G.p, rows * rows, s);
            gram = nullptr;
        }
        o = factor_from_gram(gram ? gram : G.p, rows, budget, s, oz);
    } else {  // thin left singular vectors from the Gram of B^T (sthosvd.cpp:91-99)
        EigWork w;
        DevBuf<double> G(cols * cols, s);
        gram_cols_f64(x, rows, cols, G.p, s);
        u64 r = 0;
        double gone = 0.0;
        std::vector<double> s2;
        DevBuf<double> V;
        if (!topk_factor(G.p, cols, budget, s, r, gone, s2, V, &o.tie)) {
            const double bv = budget.eval(budget.trace_out ? gram_trace(G.p, cols, s) : 0.0);
            const auto ev = eig_values(G.p, cols, w, s);
            s2.assign(cols, 0.0);
            for (u64 j = 0; j < cols; ++j) s2[j] = std::max(0.0, ev[j]);
            std::tie(r, gone) = pick_rank(s2, bv);
            o.tie = rank_tie(s2, r, gone, bv);
            if (r == 0) {
                r = 1;
                gone -= s2[0];
            }
            V = DevBuf<double>(cols * r, s);
            eig_vectors(w, r, V.p, s);
        }
        o.r = r;
        o.discarded = gone;
        o.U = DevBuf<double>(rows * r, s);
        gemm_nn_f64(x, rows, cols, V.p, r, o.U.p, s);
        std::vector<double> sig(r);
        for (u64 j = 0; j < r; ++j) sig[j] = std::sqrt(s2[j]);
        DevBuf<double> ds(r, s);
        ds.upload(sig.data(), r);
        scale_orthonormalize(o.U.p, rows, r, ds.p, s);
        stream_sync(s);
        fix_column_signs(o.U.p, rows, r, s);
    }
    o.next = DevBuf<double>(cols * o.r, s);
    if (ozaki_ttm_ok(rows, cols, o.r)) {
        ttm_ozaki(x, rows, cols, o.U.p, o.r, o.next.p, s, tprep.get());
    } else {
        ttm_f64(x, rows, cols, o.U.p, o.r, o.next.p, s);
        if (tprep) {  // unused: released after its kernels, in the call's stream order
            TCB_CUDA(cudaStreamWaitEvent(s, tprep->done, 0));
            tprep->exc.s = s;
            tprep->dt.s = s;
        }
    }
    return o;
}

Tucker sthosvd_device(DevBuf<double>&& owned, const double* ext, const std::vector<u64>& shape, double target,
                      const std::optional<std::vector<u64>>& order, int backend, cudaStream_t s, int finite,
                      const std::function<void(std::size_t, const double*, u64, u64)>& on_factor,
                      double norm_scale, double* norm_out, const double* gram0, const ShardComm* shard) {
    const bool sharded = shard && shard->world > 1;
    if (target < 0) throw Error("sthosvd: negative SSE target");
    const std::size_t d = shape.size();
    std::vector<u64> p = order ? *order : stable_ascending(shape);
    const bool perm_ok = valid_perm(p, d);  // checked after the finiteness test, as the reference does
    std::vector<u64> lshape = shape;  // this rank's slab: the last processed mode is local
    if (shard && perm_ok) lshape[p[d - 1]] = shard->local_extent;
    u64 n_el = 1;
    for (auto v : lshape) n_el *= v;
    const double* a = ext ? ext : owned.p;
    if (finite < 0) {
        bool fin = true;
        sum_squares(a, n_el, &fin, s);
        finite = fin ? 1 : 0;
    }
    if (!finite) throw Error("sthosvd: input contains non-finite values");
    if (!perm_ok) throw Error("sthosvd: invalid processing order");
    Tucker f;
    f.order = p;
    f.n = shape;
    f.r.assign(d, 0);
    f.trunc.assign(d, 0.0);
    f.factors.resize(d);
    bool ident = true;
    for (std::size_t i = 0; i < d; ++i) ident = ident && p[i] == i;
    DevBuf<double> x;
    const double* xp = nullptr;
    if (ident) {  // mode 0 reads the input in place
        if (ext) {
            xp = ext;
        } else {
            x = std::move(owned);
            xp = x.p;
        }
    } else {
        x = DevBuf<double>(n_el, s);
        permute_axes(a, x.p, lshape, p, s);
        owned.release();
        xp = x.p;
    }
    std::vector<u64> cur(d);
    for (std::size_t i = 0; i < d; ++i) cur[i] = lshape[p[i]];
    double remaining = target;
    for (std::size_t step = 0; step < d; ++step) {
        u64 tot = 1;
        for (auto v : cur) tot *= v;
        const u64 rows = cur[0], cols = tot / rows;
        Budget budget(remaining / static_cast<double>(d - step));
        double trace0 = 0.0;
        if (step == 0 && norm_out) {  // the norm from this Gram; target = norm_scale |A|^2 if >= 0
            if (norm_scale >= 0) budget.scale = norm_scale / static_cast<double>(d);
            budget.trace_out = &trace0;
        }
        HostTrace ht("sthosvd: mode step");
        StepOut so;
        if (sharded && step == d - 1) {  // the slabs meet: gather the projected tensor, step replicated
            const u64 full_rows = shape[p[d - 1]];
            if (rows * static_cast<u64>(shard->world) != full_rows)
                throw Error("sharded compress: slabs must split the last processed mode evenly");
            DevBuf<double> full(full_rows * cols, s);
            shard->allgather(xp, full.p, rows * cols * sizeof(double), s);
            x = std::move(full);
            xp = x.p;
            so = mode_step(xp, full_rows, cols, budget, backend, s);
        } else {
            so = mode_step(xp, rows, cols, budget, backend, s, step == 0 && ident ? gram0 : nullptr,
                           step + 1 < d ? shard : nullptr);
        }
        if (step == 0 && norm_out) {
            if (norm_scale >= 0) remaining = norm_scale * trace0;
            *norm_out = trace0;
        }
        remaining = std::max(0.0, remaining - so.discarded);
        f.trunc[p[step]] = so.discarded;
        x = std::move(so.next);
        xp = x.p;
        f.factors[p[step]] = std::move(so.U);
        f.r[p[step]] = so.r;
        if (so.tie) f.tie_modes |= 1u << p[step];
        // the factor's rows: the whole mode (the sharded last step ran on the gathered tensor)
        const u64 frows = sharded && step == d - 1 ? shape[p[d - 1]] : rows;
        if (on_factor) on_factor(p[step], f.factors[p[step]].p, frows, so.r);
        cur.erase(cur.begin());
        cur.push_back(so.r);
    }
    f.core = std::move(x);
    f.core_shape = cur;
    stream_sync(s);
    return f;
}

FactorPrep factor_prepare(const double* U, u64 n, u64 r, const std::vector<u8>& dead, bool f32, cudaStream_t s) {
    FactorPrep pp;
    for (u64 j = 0; j < r; ++j)
        if (!dead[j]) pp.live.push_back(j);
    const u64 rl = pp.live.size();
    try {
        if (rl == 0) return pp;
        if (rl > n) throw Error("factorize: more columns than rows");
        if (orth_deviation(U, n, r, pp.live, f32, s) > 1e-8)
            throw Error("factorize: input columns are not orthonormal");
        pp.V = DevBuf<double>(n * rl, s);
        pp.fl.resize(rl);
        householder(U, n, r, pp.live, pp.V.p, pp.fl.data(), s);
    } catch (...) {
        pp.err = std::current_exception();
    }
    return pp;
}

void factor_quantize(FactorQuant& q, const FactorPrep& prep, u64 n, const std::vector<double>& sn_live, bool simple,
                     cudaStream_t s) {
    const u64 rl = prep.live.size();
    q.live = prep.live;
    q.ln = sn_live;
    q.sc.assign(rl, 0.0);
    if (simple) {
        q.sc = q.ln;
    } else {
        const auto al = alpha_weights(q.ln, n);
        for (u64 j = 0; j < rl; ++j) q.sc[j] = std::sqrt(2.0 * al[j]);
    }
    q.dsc = DevBuf<double>(rl, s);
    q.dsc.upload(q.sc.data(), rl);
    q.dfl = DevBuf<signed char>(rl, s);
    q.dfl.upload(prep.fl.data(), rl);
    q.cnt = n * rl - rl * (rl + 1) / 2;
    DevBuf<double> st(q.cnt, s);
    reflector_stream(prep.V.p, n, rl, q.dsc.p, st.p, s);
    const double mx = q.cnt ? max_abs(st.p, q.cnt, s) : 0.0;
    q.k = mx > 0.0 ? 63 - std::ilogb(mx) : 0;
    q.mag = DevBuf<u64>(q.cnt, s);
    q.neg = DevBuf<u8>(q.cnt, s);
    quantize_f64(st.p, q.cnt, q.k, q.mag.p, q.neg.p, s);
}

void factor_plane_search(FactorQuant& q, const double* U, u64 n, u64 r, int core_step_log2, double cap,
                         cudaStream_t s) {
    const u64 rl = q.live.size();
    int plane = std::clamp(core_step_log2 + q.k, 0, 63);
    // The reference deepens the plane while the factor term exceeds the cap
    // (factor_codec.cpp:218-243).  Terms for a window of 4 candidate planes are
    // evaluated in one batched launch (each candidate expands every reflector:
    // a wider window cost more GPU time beside the core's encoder than the extra
    // round trip it saves); the host then replays the reference's deepening
    // decisions over them.
    std::vector<double> term_of(64, -1.0);
    double term = 0.0;
    while (true) {
        if (term_of[plane] < 0.0) {
            std::vector<int> cand;
            for (int p = plane; p >= 0 && static_cast<int>(cand.size()) < 4; --p)
                if (term_of[p] < 0.0) cand.push_back(p);
            const auto res = factor_residuals(q.mag.p, q.neg.p, q.k, n, r, q.live, q.dsc.p, U, q.dfl.p, cand, s);
            for (std::size_t c = 0; c < cand.size(); ++c) {
                double t = 0.0;
                for (u64 j = 0; j < rl; ++j) t += q.ln[j] * q.ln[j] * res[c * rl + j];
                term_of[cand[c]] = t;
            }
        }
        term = term_of[plane];
        if (term <= cap || plane == 0) break;
        const double excess = term / std::max(cap, 1e-300);
        const int stp = std::max(1, static_cast<int>(std::ceil(0.25 * std::log2(excess))));
        plane = std::max(0, plane - stp);
    }
    q.core_step = core_step_log2;
    q.plane = plane;
    q.term = term;
}

FactorEnc encode_factor_device(const double* U, u64 n, u64 r, const std::vector<u8>& dead,
                               const std::vector<double>& sn, int coder, bool simple, int core_step_log2,
                               double cap, bool f32, cudaStream_t s,
                               const std::function<void(const std::vector<signed char>&)>& on_flips,
                               FactorPrep* prep, FactorQuant* spec) {
    if (dead.size() != r || sn.size() != r) throw Error("factor encode: column metadata mismatch");
    FactorEnc out;
    out.dead = dead;
    out.slice_norms = sn;
    out.flips.assign(r, 1);
    std::vector<u64> live;
    std::vector<double> ln;
    for (u64 j = 0; j < r; ++j)
        if (!dead[j]) {
            live.push_back(j);
            ln.push_back(sn[j]);
        }
    const u64 rl = live.size();
    if (rl == 0) {
        if (on_flips) on_flips(out.flips);
        out.stream = empty_stream_section(0, 0);
        return out;
    }
    // the orthonormality check + reflectors (factor_codec.cpp:29-31, 153-200), reused
    // from a speculative preparation when it was made for the same live columns
    FactorPrep own;
    if (!prep || prep->live != live) {
        own = factor_prepare(U, n, r, dead, f32, s);
        prep = &own;
        spec = nullptr;
    }
    if (prep->err) std::rethrow_exception(prep->err);
    for (u64 j = 0; j < rl; ++j) out.flips[live[j]] = prep->fl[j];
    if (on_flips) on_flips(out.flips);
    FactorQuant ownq;
    FactorQuant* q = spec && spec->live == live && spec->ln == ln ? spec : nullptr;
    if (!q) {
        factor_quantize(ownq, *prep, n, ln, simple, s);
        q = &ownq;
    }
    if (q->core_step != core_step_log2 || q->plane < 0) {
        factor_plane_search(*q, U, n, r, core_step_log2, cap, s);
        q->finalized = false;
    }
    if (!q->finalized) factor_finalize(*q, coder, s);
    out.count = q->cnt;
    out.k = q->k;
    out.term = q->term;
    out.stream = std::move(q->stream);
    out.plane = q->plane;
    return out;
}

void factor_finalize(FactorQuant& q, int coder, cudaStream_t s) {
    const u64 cnt = q.cnt;
    PlanResult pl;  // fixed last plane: planes 63..plane in full (core_codec.cpp:328-391)
    pl.block = default_block(cnt);
    if (cnt > 0) {
        pl.last_plane = q.plane;
        pl.nplanes = 64 - q.plane;
        pl.stops.assign(2 * ((cnt + pl.block - 1) / pl.block), kFull);
    }
    q.stream = finalize_stream(q.mag.p, q.neg.p, cnt, pl, coder, cnt, s);
    q.finalized = true;
}

// Phases 2-5 of compress_impl (pipeline.cpp:77-189): storage order,
// quantisation, core plan, factors, sign fold, finalize, container.
void encode_into(Result& res, Tucker& f, const std::vector<u64>& shape, int dtype, double target,
                 double core_target, double trunc, const Params& prm, cudaStream_t s, Clock::time_point t_all,
                 u64 n_el, std::vector<std::future<FactorPrep>>* preps = nullptr, const ShardComm* shard = nullptr) {
    const std::size_t d = shape.size();
    auto t0 = Clock::now();
    // phase 2: storage order + quantisation
    std::vector<u64> storage = prm.storage_order ? *prm.storage_order : stable_ascending(f.core_shape);
    if (!valid_perm(storage, d)) throw Error("compress: invalid storage order");
    std::vector<u64> cs(d);
    for (std::size_t i = 0; i < d; ++i) cs[i] = f.core_shape[storage[i]];
    u64 nc = 1;
    for (auto v : cs) nc *= v;
    DevBuf<double> core_s(nc, s);
    permute_axes(f.core.p, core_s.p, f.core_shape, storage, s);
    f.core.release();
    // vectorize::OrderMap::build (pipeline.cpp:87): null for the lexicographic default
    const DevBuf<u64> vorder = order_map_device(prm.method, cs, s);
    if (prm.f32) {  // the float core of the reference
        DevBuf<float> cf(nc, s);
        ingest_cast_f32(core_s.p, 9, nc, cf.p, s);
        ingest_cast(cf.p, 8, nc, core_s.p, s);
    }
    bool core_finite = true;
    HostTrace ht_q("encode: max + quantize launch");
    const double mx = max_abs_finite(core_s.p, nc, &core_finite, s);
    if (!core_finite) throw Error("quantize: non-finite core values");
    const bool zero = mx == 0.0;
    const int k = zero ? 0 : 63 - std::ilogb(mx);
    res.core_k = k;
    DevBuf<u64> mag(nc, s);
    DevBuf<u8> neg(nc, s);
    std::vector<double> sn_flat;
    u64 sum_ext = 0;
    for (auto v : cs) sum_ext += v;
    // the slice norms (serial per slice) feed only the factor weights: on a worker
    // stream, overlapping the core plan, when the encode runs concurrently
    const bool par_sn = d > 1 && !prof_enabled();
    std::shared_future<void> sn_ready;
    if (!zero) {
        quantize_f64(core_s.p, nc, k, mag.p, neg.p, s, vorder.p);
        if (par_sn) {
            const int dev = cur_device();
            cudaStream_t side = Workers::get().stream(dev, static_cast<int>(d) + 1);
            EventHandle q;
            TCB_CUDA(cudaEventRecord(q.e, s));
            TCB_CUDA(cudaStreamWaitEvent(side, q.e, 0));
            const double scale = std::ldexp(1.0, -2 * k);
            auto task = std::make_shared<std::packaged_task<void()>>([&, side, dev, scale, sum_ext] {
                TCB_CUDA(cudaSetDevice(dev));
                DevBuf<double> dsn(sum_ext, side);
                slice_norms(mag.p, cs, scale, dsn.p, side, vorder.p);
                sn_flat = dsn.to_host();
            });
            sn_ready = task->get_future().share();
            Workers::get().submit([task] { (*task)(); });
        } else {
            DevBuf<double> dsn(sum_ext, s);
            slice_norms(mag.p, cs, std::ldexp(1.0, -2 * k), dsn.p, s, vorder.p);
            sn_flat = dsn.to_host();
        }
    }
    struct SnJoin {  // the slice-norm task reads mag / cs / vorder: join before they unwind
        std::shared_future<void>& f;
        ~SnJoin() {
            if (f.valid()) f.wait();
        }
    } sn_join{sn_ready};
    // core_s is read by nothing after the quantisation kernel (stream-ordered free)
    core_s.release();
    ht_q.stop();
    res.times.quantize = ms_since(t0);
    const u64 block = prm.block ? prm.block : default_block(zero ? 0 : nc);

    // header (container.hpp:59-82)
    W w;
    for (char c : {'T', 'K', 'C', '1'}) w.u8v(static_cast<u8>(c));
    w.u8v(1);
    w.u8v(static_cast<u8>(dtype));
    w.u8v(prm.f32 ? 1 : 0);
    w.u8v(static_cast<u8>(d));
    w.u8v(static_cast<u8>(prm.coder));
    w.u8v(static_cast<u8>(prm.method));
    w.u8v(static_cast<u8>((zero ? 1 : 0) | (prm.split ? 2 : 0) | (prm.simple ? 4 : 0)));
    w.u8v(0);
    for (auto v : shape) w.u64v(v);
    for (auto v : f.r) w.u64v(v);
    for (auto v : f.order) w.u8v(static_cast<u8>(v));
    for (auto v : storage) w.u8v(static_cast<u8>(v));
    w.u32v(static_cast<u32>(k));
    w.u64v(block);
    w.f64v(prm.rtmss);
    w.f64v(target);
    w.f64v(res.norm_sq);
    w.f64v(trunc);

    if (zero) {
        res.estimate = trunc;
        w.f64v(0.0);
        w.f64v(trunc);
        res.container = HostBytes::from(w.b);
        res.times.total = ms_since(t_all);
        return;
    }

    std::vector<u64> mode_of(d);
    for (std::size_t ax = 0; ax < d; ++ax) mode_of[ax] = f.order[storage[ax]];
    std::vector<std::vector<double>> sn_mode(d);
    std::once_flag sn_once;
    auto need_sn = [&] {  // the slice norms by mode, once they exist
        std::call_once(sn_once, [&] {
            if (sn_ready.valid()) sn_ready.get();
            u64 o = 0;
            for (std::size_t ax = 0; ax < d; ++ax) {
                sn_mode[mode_of[ax]].assign(sn_flat.begin() + o, sn_flat.begin() + o + cs[ax]);
                o += cs[ax];
            }
        });
    };

    // phases 3-4: the core plan on `s`; meanwhile every factor's orthonormality
    // check + reflectors run speculatively on a worker stream (assuming no dead
    // columns, redone for the real live set if the plan kills some); then each
    // factor's plane search and stream finalisation, its column sign flips
    // published as soon as they are final so that the core's sign fold and
    // finalisation overlap the factors.  Sequential while per-stage profiling is on.
    t0 = Clock::now();
    EncodeOpts eo;
    eo.coder = prm.coder;
    eo.block = block;
    eo.split = prm.split;
    eo.shard = shard && shard->world > 1 ? shard : nullptr;
    DevBuf<u64> dec(nc, s);
    const double cap = 0.02 * target / static_cast<double>(d);
    std::vector<FactorEnc> fe(d);
    res.factor_terms.assign(d, 0.0);
    std::vector<std::vector<signed char>> flips_of(d), flips_of_core(d);
    std::vector<std::vector<u8>> dead_mode(d);
    int core_step = 0;
    const bool par = d > 1 && !prof_enabled();
    std::promise<void> plan_ready;
    std::shared_future<void> plan_fut = plan_ready.get_future().share();
    // the core's last plane, published by the planner as soon as it is certified:
    // each factor's plane search depends only on it (and on the live columns)
    std::promise<int> lp_ready;
    std::shared_future<int> lp_fut = lp_ready.get_future().share();
    std::atomic<bool> lp_set{false};
    std::vector<std::promise<void>> flips_ready(d);
    std::vector<std::future<void>> flips_fut, done;
    // the speculative preparation's flips (every column live): final whenever the
    // plan kills no column of that mode, so the core need not wait for the worker
    std::vector<std::vector<signed char>> spec_flips(d);
    std::vector<std::promise<bool>> spec_ready(d);
    std::vector<std::shared_future<bool>> spec_fut;
    JoinAll join{done};
    struct PlanGuard {  // a throwing plan must still release the workers
        std::promise<void>& p;
        std::promise<int>& lp;
        std::atomic<bool>& lp_set;
        bool set = false;
        ~PlanGuard() {
            if (!set) p.set_exception(std::make_exception_ptr(Error("compress: core plan failed")));
            if (!lp_set.exchange(true)) lp.set_exception(std::make_exception_ptr(Error("compress: core plan failed")));
        }
    } plan_guard{plan_ready, lp_ready, lp_set};
    HostTrace ht_launch("encode: launch workers");
    if (par) {
        int dev = 0;
        TCB_CUDA(cudaGetDevice(&dev));
        EventHandle ready;
        TCB_CUDA(cudaEventRecord(ready.e, s));
        Workers& pool = Workers::get();
        for (std::size_t i = 0; i < d; ++i) {
            flips_fut.push_back(flips_ready[i].get_future());
            spec_fut.push_back(spec_ready[i].get_future().share());
            cudaStream_t si = pool.stream(dev, static_cast<int>(i));
            TCB_CUDA(cudaStreamWaitEvent(si, ready.e, 0));
            done.push_back(pool.submit([&, i, si, dev] {
                bool sent = false, spec_sent = false;
                try {
                    TCB_CUDA(cudaSetDevice(dev));
                    FactorPrep prep = preps && i < preps->size() && (*preps)[i].valid()
                                          ? (*preps)[i].get()  // made during the mode loop
                                          : factor_prepare(f.factors[i].p, f.n[i], f.r[i],
                                                           std::vector<u8>(f.r[i], 0), prm.f32, si);
                    if (!prep.err && prep.live.size() == f.r[i]) spec_flips[i] = prep.fl;
                    spec_sent = true;
                    spec_ready[i].set_value(!prep.err && prep.live.size() == f.r[i]);
                    // speculation "no dead columns": quantised stream now, plane search as
                    // soon as the core's last plane is certified
                    FactorQuant spec;
                    bool have_spec = false;
                    if (!prep.err && !prep.live.empty()) {
                        need_sn();
                        factor_quantize(spec, prep, f.n[i], sn_mode[i], prm.simple, si);
                        have_spec = true;
                        const int lp = lp_fut.get();
                        factor_plane_search(spec, f.factors[i].p, f.n[i], f.r[i], lp - k, cap, si);
                        factor_finalize(spec, prm.coder, si);
                    }
                    plan_fut.get();
                    need_sn();
                    fe[i] = encode_factor_device(
                        f.factors[i].p, f.n[i], f.r[i], dead_mode[i], sn_mode[i], prm.coder, prm.simple, core_step,
                        cap, prm.f32, si,
                        [&](const std::vector<signed char>& fl) {
                            flips_of[i] = fl;
                            sent = true;
                            flips_ready[i].set_value();
                        },
                        &prep, have_spec ? &spec : nullptr);
                } catch (...) {
                    if (!spec_sent) spec_ready[i].set_value(false);
                    if (!sent) flips_ready[i].set_exception(std::current_exception());
                    throw;
                }
            }));
        }
    }
    ht_launch.stop();
    HostTrace ht_probe("encode: probe launch");
    // speculative split probe: every full plane's entropy size on a side stream
    // (small cores only: 64 streams per block)
    std::shared_ptr<ProbeCache> probe;
    if (par && prm.split && nc <= (u64{1} << 20) && 64 * ((nc + block - 1) / block) <= 4096) {
        int dev = 0;
        TCB_CUDA(cudaGetDevice(&dev));
        cudaStream_t side = Workers::get().stream(dev, static_cast<int>(d));
        EventHandle q;
        TCB_CUDA(cudaEventRecord(q.e, s));
        TCB_CUDA(cudaStreamWaitEvent(side, q.e, 0));
        probe = probe_planes_async(mag.p, nc, block, prm.coder, side);
        eo.probe = probe.get();
    }
    ht_probe.stop();
    // The full planes above the breakpoint do not depend on the stops, the probe
    // or the dead slices: once the planner finds the breakpoint they are emitted
    // and coded on a worker stream, with the signs folded by the speculative
    // (every column live) flips.  Used when the final flips equal those.
    struct Upper {
        int p = -1;
        std::future<EmitDev> fut;
        ~Upper() {
            if (fut.valid()) fut.wait();  // the task reads this frame's buffers
        }
    } upper;
    // Off by default: on c5 the upper planes' emission competes with the probe and
    // the plane statistics for the SMs and the wait at finalisation cost more than
    // the overlap saved (542 vs 560 ms); TCB_EARLY_PLANES=1 turns it on.
    if (par && !eo.shard && d + 3 <= 8 && nc > (u64{1} << 20) && std::getenv("TCB_EARLY_PLANES")) {
        eo.on_breakpoint = [&](int p) {
            if (p >= 63 || upper.fut.valid()) return;
            const int dev = cur_device();
            cudaStream_t side = Workers::get().stream(dev, static_cast<int>(d) + 3);
            // the signs as they are now (the main stream folds them in place later)
            auto negs = std::make_shared<DevBuf<u8>>(nc, s);
            TCB_CUDA(cudaMemcpyAsync(negs->p, neg.p, nc, cudaMemcpyDeviceToDevice, s));
            EventHandle q;
            TCB_CUDA(cudaEventRecord(q.e, s));
            TCB_CUDA(cudaStreamWaitEvent(side, q.e, 0));
            upper.p = p;
            auto task = std::make_shared<std::packaged_task<EmitDev()>>([&, side, dev, p, negs]() -> EmitDev {
                TCB_CUDA(cudaSetDevice(dev));
                std::vector<signed char> fl;
                for (std::size_t i = 0; i < d; ++i)
                    if (!spec_fut[i].get()) return EmitDev{};
                for (std::size_t ax = 0; ax < d; ++ax)
                    fl.insert(fl.end(), spec_flips[mode_of[ax]].begin(), spec_flips[mode_of[ax]].end());
                negs->s = side;
                sign_fold(negs->p, cs, fl, side, vorder.p);
                EmitDev r = emit_planes_device(mag.p, negs->p, nc, block, p + 1, 63, nullptr, prm.coder, side);
                stream_sync(side);
                return r;
            });
            upper.fut = task->get_future();
            Workers::get().submit([task] { (*task)(); });
        };
    }
    PlanResult plan;
    {
        HostTrace ht("encode: core plan");
        if (par)
            eo.on_last_plane = [&](int lp) {
                if (!lp_set.exchange(true)) lp_ready.set_value(lp);
            };
        plan = plan_stream(mag.p, nc, std::ldexp(core_target, 2 * k), eo, dec.p, s);
    }
    res.core_last_plane = plan.last_plane;
    res.uncertified += plan.fallbacks;
    res.times.core = ms_since(t0);
    std::vector<u8> dead_flat;
    {
        HostTrace ht("encode: dead slices");
        dead_flat = dead_slices(dec.p, cs, s, vorder.p);
    }
    {
        u64 o = 0;
        for (std::size_t ax = 0; ax < d; ++ax) {
            dead_mode[mode_of[ax]].assign(dead_flat.begin() + o, dead_flat.begin() + o + cs[ax]);
            o += cs[ax];
        }
    }
    core_step = plan.last_plane - k;
    plan_guard.set = true;
    plan_ready.set_value();
    t0 = Clock::now();
    if (par) {
        HostTrace ht("encode: wait factor flips");
        for (std::size_t i = 0; i < d; ++i) {
            bool all_live = true;
            for (u8 v : dead_mode[i]) all_live = all_live && v == 0;
            if (all_live && spec_fut[i].get()) {
                flips_of_core[i] = spec_flips[i];  // identical to what the worker will publish
            } else {
                flips_fut[i].get();  // rethrows a factor's early error (join waits for the rest)
                flips_of_core[i] = flips_of[i];
            }
        }
    } else {
        need_sn();
        for (std::size_t i = 0; i < d; ++i)
            fe[i] = encode_factor_device(f.factors[i].p, f.n[i], f.r[i], dead_mode[i], sn_mode[i], prm.coder,
                                         prm.simple, core_step, cap, prm.f32, s,
                                         [&](const std::vector<signed char>& fl) { flips_of[i] = fl; });
        flips_of_core = flips_of;
    }

    // sign fold + finalize (pipeline.cpp:161-176)
    const auto t1 = Clock::now();
    std::vector<signed char> flips_axis;
    for (std::size_t ax = 0; ax < d; ++ax)
        flips_axis.insert(flips_axis.end(), flips_of_core[mode_of[ax]].begin(), flips_of_core[mode_of[ax]].end());
    sign_fold(neg.p, cs, flips_axis, s, vorder.p);
    u64 count = 1;
    for (auto v : f.r) count *= v;
    StreamParts core_stream;
    double ach = 0.0;
    {
        HostTrace ht("encode: core finalize+sum");
        // achieved_sse_int, accumulated backward (core_codec.cpp:405-411): needs only the
        // magnitudes and the plan's decoded values, so it runs beside the finalisation
        std::future<double> ach_fut;
        if (par) {
            const int dev = cur_device();
            cudaStream_t side = Workers::get().stream(dev, static_cast<int>(d) + 2);
            EventHandle q;
            TCB_CUDA(cudaEventRecord(q.e, s));
            TCB_CUDA(cudaStreamWaitEvent(side, q.e, 0));
            auto task = std::make_shared<std::packaged_task<double()>>([&, side, dev] {
                TCB_CUDA(cudaSetDevice(dev));
                return exact_backward_sum(kExDiff, 0, mag.p, dec.p, nc, side);
            });
            ach_fut = task->get_future();
            Workers::get().submit([task] { (*task)(); });
        }
        struct Join {
            std::future<double>& f;
            ~Join() {
                if (f.valid()) f.wait();
            }
        } join_ach{ach_fut};
        EmitDev up;
        std::function<EmitDev*()> get_up;
        if (upper.fut.valid())
            get_up = [&]() -> EmitDev* {
                HostTrace hu("encode: wait upper planes");
                up = upper.fut.get();
                bool ok = upper.p == plan.last_plane && up.body.p != nullptr;
                for (std::size_t i = 0; ok && i < d; ++i) ok = flips_of_core[i] == spec_flips[i];
                return ok ? &up : nullptr;
            };
        core_stream = finalize_stream_parts(mag.p, neg.p, nc, plan, prm.coder, count, s, eo.shard, get_up);
        ach = par ? ach_fut.get() : exact_backward_sum(kExDiff, 0, mag.p, dec.p, nc, s);
    }
    res.times.core += ms_since(t1);
    {
        HostTrace ht("encode: wait factors");
        for (auto& fu : done) fu.get();
    }
    for (std::size_t i = 0; i < d; ++i) res.factor_terms[i] = fe[i].term;
    res.times.factor = ms_since(t0);
    if (eo.shard && eo.shard->rank != 0) {  // rank 0 writes the container
        res.times.total = ms_since(t_all);
        return;
    }
    res.core_quant = std::ldexp(ach, -2 * k);
    double est = trunc + res.core_quant;
    for (double v : res.factor_terms) est += v;
    res.estimate = est;
    w.f64v(res.core_quant);
    w.f64v(est);

    t0 = Clock::now();
    std::vector<std::vector<u8>> fsec(d);
    for (std::size_t i = 0; i < d; ++i) {
        W fw;
        const auto& fi = fe[i];
        const std::size_t r = fi.slice_norms.size();
        for (std::size_t j = 0; j < r; j += 8) {
            u8 bits = 0;
            for (std::size_t q = 0; q < 8 && j + q < r; ++q)
                if (fi.dead[j + q]) bits |= static_cast<u8>(1u << q);
            fw.u8v(bits);
        }
        for (double v : fi.slice_norms) fw.f64v(v);
        fw.u32v(static_cast<u32>(fi.k));
        fw.u64v(fi.count);
        fw.raw(fi.stream);
        w.u64v(fw.b.size());
        w.raw(fw.b);
    }
    // the core section's body goes from the device straight into its place
    const u64 core_len = core_stream.head.size() + core_stream.body_size;
    w.u64v(core_len);
    w.raw(core_stream.head);
    res.container = HostBytes(w.b.size() + core_stream.body_size);
    std::memcpy(res.container.data(), w.b.data(), w.b.size());
    if (core_stream.body_size)
        TCB_CUDA(cudaMemcpyAsync(res.container.data() + w.b.size(), core_stream.body.p, core_stream.body_size,
                                 cudaMemcpyDeviceToHost, s));
    stream_sync(s);
    res.times.serialize = ms_since(t0);
    res.times.total = ms_since(t_all);
    res.peak_alloc = 2 * n_el * 8 + nc * 9 + res.container.size() * 2;
}
namespace {
thread_local int g_force_norm_pass = 0;
struct ForceNormPass {
    ForceNormPass() { ++g_force_norm_pass; }
    ~ForceNormPass() { --g_force_norm_pass; }
};
bool norm_pass_forced() {
    if (g_force_norm_pass > 0) return true;
    const char* e = std::getenv("TCB_NORM_PASS");  // debugging: the separate norm pass
    return e && *e && *e != '0';
}
}  // namespace

Result compress_device(const void* device_bytes, u64 nbytes, int dtype, const std::vector<u64>& shape,
                       const Params& prm, cudaStream_t s, const double* gram0, const ShardComm* shard,
                       DevBuf<double>* precast) {
    const auto t_all = Clock::now();
    Result res;
    const std::size_t d = shape.size();
    if (d == 0 || d > 8) throw Error("compress: tensor order must be between 1 and 8");
    u64 n_el = 1;
    for (auto v : shape) {
        if (v == 0) throw Error("tensor: zero-sized mode");
        n_el *= v;
    }
    res.original_bytes = n_el * dtype_size(dtype);
    const bool sharded = shard && shard->world > 1;
    if (shard) {  // this rank holds a slab of the last processed mode: local element count
        const std::vector<u64> pp = prm.mode_order ? *prm.mode_order : stable_ascending(shape);
        if (!valid_perm(pp, d)) throw Error("sthosvd: invalid processing order");
        n_el = n_el / shape[pp[d - 1]] * shard->local_extent;
    }
    if (nbytes != n_el * dtype_size(dtype))
        throw Error("ingest: buffer holds " + std::to_string(nbytes) + " bytes, expected " +
                    std::to_string(n_el * dtype_size(dtype)));
    if (prm.target_re && prm.target_sse)
        throw Error("compress: relative-error and SSE targets are mutually exclusive");
    if (!prm.target_re && !prm.target_sse) throw Error("compress: no error target given");

    // ingest (container.cpp:69-94): the internal tensor in double; with
    // internal_float32 the values are first rounded to float as the reference does
    // fp64 input (container::Dtype 9) is used in place: no ingest copy
    const bool direct = !prm.f32 && dtype == 9 && reinterpret_cast<uintptr_t>(device_bytes) % 16 == 0;
    // fp64 in place or an fp32 source: |A|^2 is read off the first mode's Gram
    // (its trace: every unfolding holds every element), so no separate norm pass
    // precedes the mode loop; a non-finite trace falls back to the element scan
    // (the reference's non-finite error, or a huge finite input)
    // (for an fp32 source only when the first Gram is the Ozaki one, whose diagonal
    // is a fixed-tree fp64 row sum of squares; the DMMA Gram's split-K diagonal is
    // ~1e-13 off the exact sum, where the element scan is within 1e-15)
    const bool src_f32 = dtype == 8;
    bool first_oz = false;
    if (src_f32 && !shape.empty()) {
        const std::vector<u64> pp = prm.mode_order ? *prm.mode_order : stable_ascending(shape);
        if (valid_perm(pp, d) && shape[pp[0]] > 0) first_oz = ozaki_gram_ok(shape[pp[0]], n_el / shape[pp[0]]);
    }
    const bool norm_from_gram = !prm.f32 && (direct || (src_f32 && first_oz)) && !norm_pass_forced();
    DevBuf<double> a;
    bool finite = true;
    if (direct && norm_from_gram) {
        res.norm_sq = 0.0;  // set after the first mode step
    } else if (src_f32 && norm_from_gram) {
        if (precast && precast->p && precast->n == n_el) {
            a = std::move(*precast);
        } else {
            a = DevBuf<double>(n_el, s);
            ingest_cast(device_bytes, dtype, n_el, a.p, s);
            gram0 = nullptr;  // computed for a cast that did not arrive
        }
        res.norm_sq = 0.0;  // set after the first mode step
    } else if (direct) {
        res.norm_sq = sum_squares(static_cast<const double*>(device_bytes), n_el, &finite, s);
    } else if (prm.f32) {
        a = DevBuf<double>(n_el, s);
        DevBuf<float> af(n_el, s);
        ingest_cast_f32(device_bytes, dtype, n_el, af.p, s);
        ingest_cast(af.p, 8, n_el, a.p, s);
        res.norm_sq = sum_squares(af.p, n_el, &finite, s);
    } else {
        a = DevBuf<double>(n_el, s);
        ingest_cast(device_bytes, dtype, n_el, a.p, s);
        res.norm_sq = sum_squares(a.p, n_el, &finite, s);
    }
    if (dtype == 6 || dtype == 7) res.precision_loss = ingest_precision_loss(device_bytes, dtype, n_el, s);
    if (sharded && !norm_from_gram) {  // global norm, finite flag and precision flag
        DevBuf<double> st(3, s);
        const double h[3] = {res.norm_sq, finite ? 0.0 : 1.0, res.precision_loss ? 1.0 : 0.0};
        st.upload(h, 3);
        shard->allreduce_sum_f64(st.p, 3, s);
        const auto g = st.to_host();
        res.norm_sq = g[0];
        finite = g[1] == 0.0;
        res.precision_loss = g[2] != 0.0;
    }
    double target;
    if (prm.target_re) {
        if (*prm.target_re < 0) throw Error("budget: negative relative-error target");
        target = *prm.target_re * *prm.target_re * res.norm_sq;
    } else {
        target = *prm.target_sse;
    }
    if (target < 0) throw Error("budget: negative SSE target");
    if (prm.rtmss < 0 || prm.rtmss > 1) throw Error("budget: rtmss outside [0, 1]");
    res.target_sse = target;
    // with the norm from the first Gram: target = norm_scale |A|^2 (relative
    // target), else fixed; either way the norm is reported from the trace
    double norm_scale = -1.0, norm_trace = 0.0;
    if (norm_from_gram) norm_scale = prm.target_re ? prm.rtmss * *prm.target_re * *prm.target_re : -1.0;

    auto t0 = Clock::now();
    // each factor's orthonormality check + reflectors start on its worker stream
    // as soon as its mode step is done, overlapping the rest of the mode loop
    const std::size_t dd = shape.size();
    std::vector<std::future<FactorPrep>> preps(dd);
    struct PrepJoin {  // no prep task may outlive this frame
        std::vector<std::future<FactorPrep>>& v;
        ~PrepJoin() {
            for (auto& x : v)
                if (x.valid()) x.wait();
        }
    } prep_join{preps};
    std::function<void(std::size_t, const double*, u64, u64)> on_factor;
    static const bool no_early_prep = [] {  // debugging: factor prep after the mode loop
        const char* e = std::getenv("TCB_NO_EARLY_PREP");
        return e && *e && *e != '0';
    }();
    if (dd > 1 && !prof_enabled() && !no_early_prep) {
        int dev = 0;
        TCB_CUDA(cudaGetDevice(&dev));
        on_factor = [&, dev](std::size_t mode, const double* U, u64 n, u64 r) {
            cudaStream_t si = Workers::get().stream(dev, static_cast<int>(mode));
            auto ready = std::make_shared<EventHandle>();
            TCB_CUDA(cudaEventRecord(ready->e, s));
            TCB_CUDA(cudaStreamWaitEvent(si, ready->e, 0));
            // the task works on its own copy of U (the Tucker may unwind first on an error)
            auto Uc = std::make_shared<DevBuf<double>>(n * r, si);
            if (n * r)
                TCB_CUDA(cudaMemcpyAsync(Uc->p, U, n * r * sizeof(double), cudaMemcpyDeviceToDevice, si));
            auto task = std::make_shared<std::packaged_task<FactorPrep()>>([Uc, n, r, f32 = prm.f32, si, dev, ready] {
                TCB_CUDA(cudaSetDevice(dev));
                FactorPrep pp = factor_prepare(Uc->p, n, r, std::vector<u8>(r, 0), f32, si);
                return pp;
            });
            preps[mode] = task->get_future();
            Workers::get().submit([task] { (*task)(); });
        };
    }
    Tucker f;
    try {
        f = sthosvd_device(std::move(a), direct ? static_cast<const double*>(device_bytes) : nullptr, shape,
                           prm.rtmss * target, prm.mode_order, prm.backend, s, finite ? 1 : 0, on_factor,
                           norm_scale, norm_from_gram ? &norm_trace : nullptr,
                           direct || (src_f32 && norm_from_gram) ? gram0 : nullptr, shard);
    } catch (const TraceNonFinite&) {  // scan the elements: the reference error, or a norm pass rerun
        bool fin = true;
        if (direct) sum_squares(static_cast<const double*>(device_bytes), n_el, &fin, s);
        else sum_squares(static_cast<const float*>(device_bytes), n_el, &fin, s);
        if (sharded) {  // every rank sees the same trace, so every rank is here: agree on the verdict
            DevBuf<double> f(1, s);
            const double h = fin ? 0.0 : 1.0;
            f.upload(&h, 1);
            shard->allreduce_sum_f64(f.p, 1, s);
            fin = f.to_host()[0] == 0.0;
        }
        if (!fin) throw Error("sthosvd: input contains non-finite values");
        ForceNormPass force;
        return compress_device(device_bytes, nbytes, dtype, shape, prm, s, gram0, shard);
    }
    if (norm_from_gram) {
        res.norm_sq = norm_trace;
        if (prm.target_re) {
            target = *prm.target_re * *prm.target_re * res.norm_sq;
            res.target_sse = target;
        }
    }
    double trunc = 0;
    for (double v : f.trunc) trunc += v;
    double core_target = target - trunc;
    if (core_target < 0) core_target = 0;
    res.times.sthosvd = ms_since(t0);
    res.trunc = trunc;
    res.ranks = f.r;
    res.rank_tie_modes = f.tie_modes;

    // every rank encodes its share of the core's blocks (the factorisation is replicated)
    encode_into(res, f, shape, dtype, target, core_target, trunc, prm, s, t_all, n_el, &preps, shard);
    return res;
}

Result encode_tucker_device(Tucker& f, int dtype, double norm_sq, double target, const Params& prm, cudaStream_t s,
                            const ShardComm* shard) {
    const auto t_all = Clock::now();
    Result res;
    const std::vector<u64> shape = f.n;
    u64 n_el = 1;
    for (auto v : shape) n_el *= v;
    res.original_bytes = n_el * dtype_size(dtype);
    res.norm_sq = norm_sq;
    res.target_sse = target;
    double trunc = 0;
    for (double v : f.trunc) trunc += v;
    double core_target = target - trunc;
    if (core_target < 0) core_target = 0;
    res.trunc = trunc;
    res.ranks = f.r;
    encode_into(res, f, shape, dtype, target, core_target, trunc, prm, s, t_all, n_el, nullptr, shard);
    return res;
}


}  // namespace tcb
