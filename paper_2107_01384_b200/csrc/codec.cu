// Bit-plane codec kernels: the bit-exact half of the compress path.
//
// Statistics (core_codec.cpp:120-171, error_model.cpp:34-72): every term is
// computed with separately rounded __dmul_rn/__dsub_rn exactly as the
// reference's x86-64 build (no FMA contraction), summed in double-double
// (error ~2^-104) together with a rigorous bound on the reference's serial
// rounding error, so the host can certify each breakpoint/stop decision and
// fall back to the serial replay kernels below only when it cannot.
//
// Emission (core_codec.cpp:120-171, entropy.cpp:22-239): one CTA per
// (plane, block) stream classifies positions with CTA-wide scans, writes the
// zero-run symbols and the MSB-first raw bits; the adaptive range coder then
// runs one thread per stream; payloads are compacted in stream order.
#include <algorithm>
#include <mutex>
#include <cfloat>

#include "codec.cuh"

namespace tcb {

namespace {

__device__ __forceinline__ int top_bit(u64 m) { return m ? 63 - __clzll(static_cast<long long>(m)) : -1; }

// residual^2 of a significant coefficient with planes >= p known (core_codec.cpp:20-30)
__device__ __forceinline__ double sig2(u64 m, int p) {
    if (p == 0) return 0.0;
    const u64 low = m & ((u64{1} << p) - 1);
    const double r = __dsub_rn(__ull2double_rn(low), __ull2double_rn(u64{1} << (p - 1)));
    return __dmul_rn(r, r);
}
__device__ __forceinline__ double insig2(u64 m) {
    const double v = __ull2double_rn(m);
    return __dmul_rn(v, v);
}
__device__ __forceinline__ double trail_gain(u64 m, int p) { return __dsub_rn(sig2(m, p + 1), sig2(m, p)); }
__device__ __forceinline__ double lead_gain(u64 m, int p) { return __dsub_rn(insig2(m), sig2(m, p)); }

struct DD {
    double hi, lo;
};
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
    s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
__device__ __forceinline__ DD dd_add(DD x, double t) {
    double s, e;
    two_sum(x.hi, t, s, e);
    e = __dadd_rn(e, x.lo);
    DD r;
    two_sum(s, e, r.hi, r.lo);
    return r;
}
__device__ __forceinline__ DD dd_add(DD x, DD y) {
    double s, e;
    two_sum(x.hi, y.hi, s, e);
    e = __dadd_rn(e, __dadd_rn(x.lo, y.lo));
    DD r;
    two_sum(s, e, r.hi, r.lo);
    return r;
}

__device__ __forceinline__ double recal_term(u64 m, int plane) {
    double r;
    if (plane >= 64 || (m >> plane) == 0) r = __ull2double_rn(m);
    else if (plane == 0) r = 0.0;
    else r = __dsub_rn(__ull2double_rn(m & ((u64{1} << plane) - 1)), __ull2double_rn(u64{1} << (plane - 1)));
    return __dmul_rn(r, r);
}

__device__ __forceinline__ double sum_term(SumKind k, const u64* m, const u64* dec, u64 i, int plane) {
    switch (k) {
        case SumKind::sq_backward: return insig2(m[i]);
        case SumKind::recal_backward: return recal_term(m[i], plane);
        default: {
            const double r = __dsub_rn(__ull2double_rn(m[i]), __ull2double_rn(dec[i]));
            return __dmul_rn(r, r);
        }
    }
}

constexpr int kSumThreads = 256;

__global__ void sum_kernel(SumKind kind, const u64* __restrict__ m, const u64* __restrict__ dec, u64 n, int plane,
                           SumRec* __restrict__ part) {
    __shared__ double sh[3][kSumThreads / 32];
    DD acc{0.0, 0.0};
    double w = 0.0;
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double t = sum_term(kind, m, dec, i, plane);
        acc = dd_add(acc, t);
        w = fma(fabs(t), static_cast<double>(i + 1), w);  // backward: x_i sits in i+1 partial sums
    }
    for (int o = 16; o > 0; o >>= 1) {
        DD other{__shfl_down_sync(0xffffffffu, acc.hi, o), __shfl_down_sync(0xffffffffu, acc.lo, o)};
        acc = dd_add(acc, other);
        w += __shfl_down_sync(0xffffffffu, w, o);
    }
    const int wid = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        sh[0][wid] = acc.hi;
        sh[1][wid] = acc.lo;
        sh[2][wid] = w;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        DD t{0.0, 0.0};
        double ww = 0.0;
        for (int i = 0; i < kSumThreads / 32; ++i) {
            t = dd_add(t, DD{sh[0][i], sh[1][i]});
            ww += sh[2][i];
        }
        part[blockIdx.x] = SumRec{t.hi, t.lo, ww, 0};
    }
}

// Serial replay of a backward sum (the exact-mode fallback): the CTA computes
// the terms of the next chunk into shared memory (coalesced loads) while
// thread 0 runs the dependent __dadd_rn chain over the current one from
// registers, 8 at a time -- about one add latency per element instead of one
// memory latency.
constexpr int kSerThreads = 256, kSerChunk = 2048;
__device__ double serial_sum_cta(SumKind kind, const u64* __restrict__ m, const u64* __restrict__ dec, u64 n,
                                 int plane, double (*buf)[kSerChunk]) {
    const u64 nchunk = (n + kSerChunk - 1) / kSerChunk;
    auto fill = [&](u64 c, int b) {  // chunk c = indices [n - (c+1) C, n - c C), stored in descending order
        const u64 hi = n - c * kSerChunk;
        for (int q = threadIdx.x; q < kSerChunk; q += blockDim.x)
            buf[b][q] = static_cast<u64>(q) < hi ? sum_term(kind, m, dec, hi - 1 - q, plane) : 0.0;
    };
    double s = 0.0;
    if (nchunk) fill(0, 0);
    __syncthreads();
    for (u64 c = 0; c < nchunk; ++c) {
        const int b = static_cast<int>(c & 1);
        if (c + 1 < nchunk) fill(c + 1, b ^ 1);
        if (threadIdx.x == 0) {
            const u64 hi = n - c * kSerChunk;
            const int cnt = static_cast<int>(hi < kSerChunk ? hi : kSerChunk);
            for (int q0 = 0; q0 < cnt; q0 += 8) {
                double t[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) t[u] = buf[b][q0 + u];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (q0 + u < cnt) s = __dadd_rn(s, t[u]);
            }
        }
        __syncthreads();
    }
    return s;
}

__global__ void __launch_bounds__(kSerThreads) sum_serial_kernel(SumKind kind, const u64* __restrict__ m,
                                                                const u64* __restrict__ dec, u64 n, int plane,
                                                                double* out) {
    __shared__ double buf[2][kSerChunk];
    const double s = serial_sum_cta(kind, m, dec, n, plane, buf);
    if (threadIdx.x == 0) *out = s;
}

// several independent serial sums at once (one CTA each): the exact planner's
// initial sum and every plane's recalibration sum, in the time of one
__global__ void __launch_bounds__(kSerThreads) sum_serial_multi_kernel(const int* __restrict__ kinds,
                                                                      const int* __restrict__ planes,
                                                                      const u64* __restrict__ m, u64 n,
                                                                      double* __restrict__ out) {
    __shared__ double buf[2][kSerChunk];
    const double s = serial_sum_cta(static_cast<SumKind>(kinds[blockIdx.x]), m, nullptr, n, planes[blockIdx.x], buf);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// ---------------------------------------------------------------- per-plane stats
constexpr int kStatThreads = 256;
constexpr int kStatPer = 8;
constexpr u64 kChunk = static_cast<u64>(kStatThreads) * kStatPer;

struct Partial {
    double lhi, llo, lw, thi, tlo, tw;
    u64 nlead, nones, ntrail;
};

__global__ void stats_kernel(const u64* __restrict__ m, u64 n, u64 block, u64 cpb, int p_hi,
                             Partial* __restrict__ part) {
    const int p = p_hi - static_cast<int>(blockIdx.y);
    const u64 b = blockIdx.x / cpb, j = blockIdx.x % cpb;
    const u64 blo = b * block, bhi = min(n, blo + block);
    const u64 lo = blo + j * kChunk, hi = min(bhi, lo + kChunk);
    DD L{0.0, 0.0}, T{0.0, 0.0};
    double lw = 0.0, tw = 0.0;
    u64 nl = 0, no = 0, nt = 0;
    for (u64 i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const u64 v = m[i];
        const int tb = top_bit(v);
        const double rest = static_cast<double>(bhi - i);  // >= #terms from here to the block end
        if (tb > p) {
            const double t = trail_gain(v, p);
            T = dd_add(T, t);
            tw = fma(fabs(t), rest, tw);
            ++nt;
        } else {
            ++nl;
            if (tb == p) {
                const double t = lead_gain(v, p);
                L = dd_add(L, t);
                lw = fma(fabs(t), rest, lw);
                ++no;
            }
        }
    }
    __shared__ Partial sh[kStatThreads / 32];
    for (int o = 16; o > 0; o >>= 1) {
        L = dd_add(L, DD{__shfl_down_sync(0xffffffffu, L.hi, o), __shfl_down_sync(0xffffffffu, L.lo, o)});
        T = dd_add(T, DD{__shfl_down_sync(0xffffffffu, T.hi, o), __shfl_down_sync(0xffffffffu, T.lo, o)});
        lw += __shfl_down_sync(0xffffffffu, lw, o);
        tw += __shfl_down_sync(0xffffffffu, tw, o);
        nl += __shfl_down_sync(0xffffffffu, nl, o);
        no += __shfl_down_sync(0xffffffffu, no, o);
        nt += __shfl_down_sync(0xffffffffu, nt, o);
    }
    const int wid = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sh[wid] = Partial{L.hi, L.lo, lw, T.hi, T.lo, tw, nl, no, nt};
    __syncthreads();
    if (threadIdx.x == 0) {
        DD l{0.0, 0.0}, t{0.0, 0.0};
        Partial r{};
        for (int i = 0; i < kStatThreads / 32; ++i) {
            l = dd_add(l, DD{sh[i].lhi, sh[i].llo});
            t = dd_add(t, DD{sh[i].thi, sh[i].tlo});
            r.lw += sh[i].lw;
            r.tw += sh[i].tw;
            r.nlead += sh[i].nlead;
            r.nones += sh[i].nones;
            r.ntrail += sh[i].ntrail;
        }
        r.lhi = l.hi;
        r.llo = l.lo;
        r.thi = t.hi;
        r.tlo = t.lo;
        part[(static_cast<u64>(blockIdx.y) * gridDim.x) + blockIdx.x] = r;
    }
}

__global__ void stats_combine(const Partial* __restrict__ part, u64 nb, u64 cpb, int nplanes,
                              PlaneBlockRec* __restrict__ out, u64 n, u64 block) {
    const u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= nb * static_cast<u64>(nplanes)) return;
    const u64 pl = idx / nb, b = idx % nb;
    DD l{0.0, 0.0}, t{0.0, 0.0};
    PlaneBlockRec r{};
    for (u64 j = 0; j < cpb; ++j) {
        const Partial& q = part[pl * nb * cpb + b * cpb + j];
        l = dd_add(l, DD{q.lhi, q.llo});
        t = dd_add(t, DD{q.thi, q.tlo});
        r.lead.wabs += q.lw;
        r.trail.wabs += q.tw;
        r.nlead += q.nlead;
        r.nones += q.nones;
        r.ntrail += q.ntrail;
    }
    r.lead.hi = l.hi;
    r.lead.lo = l.lo;
    r.lead.nterms = r.nones;
    r.trail.hi = t.hi;
    r.trail.lo = t.lo;
    r.trail.nterms = r.ntrail;
    (void)n;
    (void)block;
    out[idx] = r;
}

// serial replay of build_block's sums for every block of one plane (one thread per block)
constexpr int kStatChunk = 1024;
// Exact per-block plane statistics (serial sums in position order): one CTA per
// block; the CTA classifies a chunk and stages the lead / trail gains in shared
// memory (zero where a position does not contribute: x + 0 = x exactly) while
// thread 0 replays both chains over the previous chunk; counts are parallel.
__global__ void __launch_bounds__(kSerThreads) stats_serial_kernel(const u64* __restrict__ m, u64 n, u64 block,
                                                                  u64 nb, int p_hi, PlaneBlockRec* __restrict__ out) {
    const int p = p_hi - static_cast<int>(blockIdx.y);
    __shared__ double lg[2][kStatChunk], tg[2][kStatChunk];
    __shared__ unsigned long long cnt_s[3];
    const u64 b = blockIdx.x;
    if (b >= nb) return;
    const u64 lo = b * block, hi = min(n, lo + block);
    const u64 len = hi - lo, nchunk = (len + kStatChunk - 1) / kStatChunk;
    if (threadIdx.x < 3) cnt_s[threadIdx.x] = 0;
    u64 my_nl = 0, my_no = 0, my_nt = 0;
    auto fill = [&](u64 c, int bb) {
        for (int q = threadIdx.x; q < kStatChunk; q += blockDim.x) {
            const u64 i = lo + c * kStatChunk + q;
            double l = 0.0, t = 0.0;
            if (i < hi) {
                const u64 v = m[i];
                const int tb = top_bit(v);
                if (tb > p) {
                    t = trail_gain(v, p);
                    ++my_nt;
                } else {
                    ++my_nl;
                    if (tb == p) {
                        l = lead_gain(v, p);
                        ++my_no;
                    }
                }
            }
            lg[bb][q] = l;
            tg[bb][q] = t;
        }
    };
    double l = 0.0, t = 0.0;
    if (nchunk) fill(0, 0);
    __syncthreads();
    for (u64 c = 0; c < nchunk; ++c) {
        const int bb = static_cast<int>(c & 1);
        if (c + 1 < nchunk) fill(c + 1, bb ^ 1);
        if (threadIdx.x == 0) {
            const u64 rem = len - c * kStatChunk;
            const int cnt = static_cast<int>(rem < kStatChunk ? rem : kStatChunk);
            for (int q0 = 0; q0 < cnt; q0 += 8) {
                double a[8], e[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    a[u] = lg[bb][q0 + u];
                    e[u] = tg[bb][q0 + u];
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (q0 + u < cnt) {
                        l = __dadd_rn(l, a[u]);
                        t = __dadd_rn(t, e[u]);
                    }
            }
        }
        __syncthreads();
    }
    atomicAdd(&cnt_s[0], static_cast<unsigned long long>(my_nl));
    atomicAdd(&cnt_s[1], static_cast<unsigned long long>(my_no));
    atomicAdd(&cnt_s[2], static_cast<unsigned long long>(my_nt));
    __syncthreads();
    if (threadIdx.x != 0) return;
    const u64 nl = cnt_s[0], no = cnt_s[1], nt = cnt_s[2];
    PlaneBlockRec r{};
    r.lead = SumRec{l, 0.0, 0.0, no};
    r.trail = SumRec{t, 0.0, 0.0, nt};
    r.nlead = nl;
    r.nones = no;
    r.ntrail = nt;
    out[static_cast<u64>(blockIdx.y) * nb + b] = r;
}

// One warp per (cum, need) pair: lanes classify 32 positions at a time and
// the warp replays the serial accumulation over them in position order.
// Serial replay of the reference's running sum over one block (the stop
// placement of core_codec.cpp:270-320): the CTA classifies a chunk of
// elements and computes their gains in parallel into shared memory, then one
// thread per pair (interval endpoint) runs the dependent __dadd_rn chain out
// of shared memory -- the loads do not depend on the chain, so each element
// costs about one add latency.  Elements are counted up to and including the
// one whose gain makes the sum reach `need`.
constexpr int kCrossThreads = 256, kCrossChunk = 4096;
__global__ void __launch_bounds__(kCrossThreads) crossing_kernel(const u64* __restrict__ m, u64 lo, u64 hi, int p,
                                                                int category, const double* __restrict__ cum0,
                                                                const double* __restrict__ need, int npairs,
                                                                u64* __restrict__ out) {
    __shared__ double tg[kCrossChunk];
    __shared__ unsigned char kd[kCrossChunk];  // 0 skip, 1 counted without term, 2 with term; 3 trailing (cat 2)
    __shared__ int live_s;
    const int k = threadIdx.x;  // serial-chain owner for pair k (threads < npairs)
    double cum = k < npairs ? cum0[k] : 0.0;
    const double nd = k < npairs ? need[k] : 0.0;
    u64 c = 0, nl = 0, nt = 0;
    bool going = k < npairs && cum < nd;
    for (u64 base = lo; base < hi; base += kCrossChunk) {
        if (threadIdx.x == 0) live_s = 0;
        __syncthreads();
        if (going) atomicOr(&live_s, 1);
        const int cnt = static_cast<int>(hi - base < kCrossChunk ? hi - base : kCrossChunk);
        for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
            const u64 v = m[base + q];
            const int tb = top_bit(v);
            int kind = 0;
            double t = 0.0;
            if (category == 0) {
                if (tb <= p) {
                    kind = tb == p ? 2 : 1;
                    if (tb == p) t = lead_gain(v, p);
                }
            } else if (category == 1) {
                if (tb > p) {
                    kind = 2;
                    t = trail_gain(v, p);
                }
            } else if (tb > p) {
                kind = 3;
                t = trail_gain(v, p);
            } else {
                kind = tb == p ? 2 : 1;
                if (tb == p) t = lead_gain(v, p);
            }
            kd[q] = static_cast<unsigned char>(kind);
            tg[q] = t;
        }
        __syncthreads();
        if (!live_s) break;
        if (going) {
            // 8 elements per step: their kinds and gains are loaded into registers
            // first, so the serial chain runs on registers, not on load latency
            for (int q0 = 0; q0 < cnt && going; q0 += 8) {
                int kk[8];
                double tt[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    kk[u] = q0 + u < cnt ? kd[q0 + u] : 0;
                    tt[u] = q0 + u < cnt ? tg[q0 + u] : 0.0;
                }
                // branch-free: kinds 0 and 1 carry a zero gain (x + 0 = x exactly), and
                // `going` is re-evaluated after every element (unchanged sums repeat the
                // previous verdict), so the chain is one add per element
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int kq = kk[u];
                    const bool counted = going && kq != 0;
                    cum = __dadd_rn(cum, tt[u]);
                    if (category == 2) {
                        nt += (counted && kq == 3) ? 1u : 0u;
                        nl += (counted && kq != 3) ? 1u : 0u;
                    } else {
                        c += counted ? 1u : 0u;
                    }
                    going = going && cum < nd;
                }
            }
        }
        __syncthreads();  // the chunk buffer is refilled next iteration
    }
    if (k < npairs) {
        if (category == 2) {
            out[2 * k] = nl;
            out[2 * k + 1] = nt;
        } else {
            out[2 * k] = c;
            out[2 * k + 1] = 0;
        }
    }
}

// ---------------------------------------------------------------- CTA scans
template <int NT>
__device__ __forceinline__ u64 cta_excl_scan(u64 v, u64* sh, u64& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u64 x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const u64 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 run = 0;
        for (int i = 0; i < NT / 32; ++i) {
            const u64 t = sh[i];
            sh[i] = run;
            run += t;
        }
        sh[NT / 32] = run;
    }
    __syncthreads();
    const u64 res = sh[w] + x - v;
    total = sh[NT / 32];
    __syncthreads();
    return res;
}

template <int NT>
__device__ __forceinline__ long long cta_excl_max(long long v, long long* sh, long long init) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = max(x, y);
    }
    long long ex = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) ex = LLONG_MIN;
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long run = init;
        for (int i = 0; i < NT / 32; ++i) {
            const long long t = sh[i];
            sh[i] = run;
            run = max(run, t);
        }
        sh[NT / 32] = run;
    }
    __syncthreads();
    const long long res = max(sh[w], ex);
    __syncthreads();
    return res;
}

// ---------------------------------------------------------------- decoded model
constexpr int kDecThreads = 256;
constexpr int kDecPer = 4;

__global__ void decode_model_kernel(const u64* __restrict__ m, u64 n, u64 block, int lp,
                                    const u64* __restrict__ stops, u64* __restrict__ dec) {
    __shared__ u64 sh[kDecThreads / 32 + 1];
    const u64 b = blockIdx.x;
    const u64 lo = b * block, hi = min(n, lo + block);
    const u64 lstop = stops[2 * b], tstop = stops[2 * b + 1];
    u64 lbase = 0, tbase = 0;
    for (u64 c0 = lo; c0 < hi; c0 += static_cast<u64>(kDecThreads) * kDecPer) {
        const u64 i0 = c0 + static_cast<u64>(threadIdx.x) * kDecPer;
        u64 v[kDecPer];
        int tb[kDecPer];
        u32 nl = 0, nt = 0;
#pragma unroll
        for (int q = 0; q < kDecPer; ++q) {
            const u64 i = i0 + q;
            v[q] = i < hi ? m[i] : 0;
            tb[q] = i < hi ? top_bit(v[q]) : -2;
            nt += tb[q] > lp;
            nl += (tb[q] <= lp && tb[q] > -2);
        }
        u64 tot;
        const u64 pre = cta_excl_scan<kDecThreads>((static_cast<u64>(nt) << 32) | nl, sh, tot);
        u64 li = lbase + (pre & 0xffffffffu), ti = tbase + (pre >> 32);
#pragma unroll
        for (int q = 0; q < kDecPer; ++q) {
            const u64 i = i0 + q;
            if (tb[q] == -2) continue;
            int pe = -1;
            if (tb[q] > lp) {
                pe = (ti++ < tstop) ? lp : lp + 1;
            } else {
                const bool within = li++ < lstop;
                if (tb[q] == lp && within) pe = lp;
            }
            u64 out = 0;
            if (pe >= 0) {
                out = pe >= 64 ? 0 : (v[q] >> pe) << pe;
                if (pe >= 1 && pe < 64) out += u64{1} << (pe - 1);
            }
            dec[i] = out;
        }
        lbase += tot & 0xffffffffu;
        tbase += tot >> 32;
    }
}

// ---------------------------------------------------------------- emission
constexpr int kEmT = 256;
constexpr int kEmPer = 4;

struct StreamDesc {
    u64 lo, hi;          // block range
    u64 lstop, tstop;
    u64 sym_off;         // into syms
    u64 raw_off;         // bit offset into raw words (multiple of 32)
    int plane;
    int pad;
};

struct StreamOut {
    u64 nsyms;    // 0 when the leading column is empty
    u64 nraw;     // raw bits
};

__global__ void __launch_bounds__(kEmT) emit_kernel(const u64* __restrict__ m, const u8* __restrict__ neg,
                                                    const StreamDesc* __restrict__ desc, u64* __restrict__ syms,
                                                    u32* __restrict__ raw, StreamOut* __restrict__ sout) {
    __shared__ u64 sh[kEmT / 32 + 1];
    __shared__ long long shm[kEmT / 32 + 1];
    const StreamDesc d = desc[blockIdx.x];
    const int p = d.plane;
    u64 lcnt = 0, tcnt = 0, rawcnt = 0, onecnt = 0;
    long long last = -1;  // lead index of the previous one
    for (u64 c0 = d.lo; c0 < d.hi; c0 += static_cast<u64>(kEmT) * kEmPer) {
        const u64 i0 = c0 + static_cast<u64>(threadIdx.x) * kEmPer;
        u64 v[kEmPer];
        int tb[kEmPer];
        u32 nl = 0, nt = 0;
#pragma unroll
        for (int q = 0; q < kEmPer; ++q) {
            const u64 i = i0 + q;
            const bool in = i < d.hi;
            v[q] = in ? m[i] : 0;
            tb[q] = in ? top_bit(v[q]) : -2;
            nt += tb[q] > p;
            nl += (tb[q] <= p && tb[q] > -2);
        }
        u64 tot;
        const u64 pre = cta_excl_scan<kEmT>((static_cast<u64>(nt) << 32) | nl, sh, tot);
        u64 li = lcnt + (pre & 0xffffffffu), ti = tcnt + (pre >> 32);
        // classify within the stops
        u32 rflag = 0, oflag = 0, nr = 0, no = 0;
        long long lastL = -1;
        u64 lidx[kEmPer];
#pragma unroll
        for (int q = 0; q < kEmPer; ++q) {
            lidx[q] = 0;
            if (tb[q] == -2) continue;
            if (tb[q] > p) {
                if (ti++ < d.tstop) {
                    rflag |= 1u << q;
                    ++nr;
                }
            } else {
                const u64 myl = li++;
                if (myl < d.lstop && tb[q] == p) {
                    oflag |= 1u << q;
                    rflag |= 1u << q;
                    ++nr;
                    ++no;
                    lidx[q] = myl;
                    lastL = static_cast<long long>(myl);
                }
            }
        }
        u64 tot2;
        const u64 pre2 = cta_excl_scan<kEmT>((static_cast<u64>(nr) << 32) | no, sh, tot2);
        const long long prevL = cta_excl_max<kEmT>(lastL, shm, last);
        u64 ri = rawcnt + (pre2 >> 32), oi = onecnt + (pre2 & 0xffffffffu);
        long long pl = prevL;
#pragma unroll
        for (int q = 0; q < kEmPer; ++q) {
            if (!(rflag >> q & 1u)) continue;
            bool bit;
            if (oflag >> q & 1u) {
                bit = neg ? neg[i0 + q] != 0 : false;
                syms[d.sym_off + oi] = static_cast<u64>(static_cast<long long>(lidx[q]) - pl - 1);
                pl = static_cast<long long>(lidx[q]);
                ++oi;
            } else {
                bit = (v[q] >> p) & 1u;
            }
            if (bit) {
                const u64 R = d.raw_off + ri;
                atomicOr(raw + (R >> 5), 1u << (8 * ((R >> 3) & 3) + (7 - (R & 7))));
            }
            ++ri;
        }
        lcnt += tot & 0xffffffffu;
        tcnt += tot >> 32;
        rawcnt += tot2 >> 32;
        onecnt += tot2 & 0xffffffffu;
        // last one index so far
        __shared__ long long shl;
        if (threadIdx.x == kEmT - 1) shl = max(prevL, lastL);
        __syncthreads();
        last = shl;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const u64 ncol = min(lcnt, d.lstop);
        StreamOut o;
        o.nraw = rawcnt;
        if (ncol > 0) {
            syms[d.sym_off + onecnt] = static_cast<u64>(static_cast<long long>(ncol) - 1 - last);
            o.nsyms = onecnt + 1;
        } else {
            o.nsyms = 0;
        }
        sout[blockIdx.x] = o;
    }
}

// ---------------------------------------------------------------- adaptive range coder
struct AcDesc {
    u64 sym_off;     // symbols
    u64 out_off;     // output byte offset (capacity 5 + 7*nsyms + 16)
    u64 model_off;   // u32 words of global scratch (global mode)
    u32 cap;         // model capacity (>= distinct symbols + 1), even
    u32 fen;         // fenwick array size (power of two >= cap + 1)
    u32 hbits;       // hash table has 1 << hbits u32 slots
    u32 pad;
};

__device__ __forceinline__ u32 hslot(u64 sym, u32 hbits) {
    return static_cast<u32>((sym * 0x9E3779B97F4A7C15ull) >> (64 - hbits));
}

constexpr u32 kAcSmemCap = 2048;  // model entries kept in shared memory (global scratch beyond)

__host__ __device__ inline u32 log2_at_least(u32 v) {
    u32 b = 5;
    while ((1u << b) < v) ++b;
    return b;
}
// model layout (u32 words): cnt[cap] | l1[cap/32+1] | l2[cap/1024+1] | hidx[1<<hb] | val[cap] (u64)
__host__ __device__ inline u64 ac_model_words(u32 cap) {
    const u64 w = cap + (cap / 32 + 1) + (cap / 1024 + 1) + (u64{1} << log2_at_least(2 * cap));
    return ((w + 1) & ~u64{1}) + 2ull * cap;
}

// One warp per stream.  The adaptive model (entropy.cpp:155-239) is resolved
// 32 symbols at a time (see the chunk comment below); all lanes then run the
// range coder redundantly (identical state) and lane 0 writes the bytes.
// Counts keep a 3-level (1 / 32 / 1024) prefix structure; halving rescales
// them with all lanes.
template <bool kShared>
__global__ void __launch_bounds__(32) ac_kernel(const u64* __restrict__ syms, const StreamOut* __restrict__ sout,
                                                const AcDesc* __restrict__ desc, const int* __restrict__ ids,
                                                int nstreams, u8* __restrict__ outbuf, u32* __restrict__ scratch,
                                                u64* __restrict__ elen, u32 smem_cap, int* __restrict__ redo) {
    extern __shared__ __align__(16) u8 ac_smem[];
    const int lane = threadIdx.x;
    const int sidx = ids ? ids[blockIdx.x] : static_cast<int>(blockIdx.x);
    if (sidx >= nstreams) return;
    const u64 ns = sout[sidx].nsyms;
    if (ns == 0) {
        if (lane == 0) elen[sidx] = 0;
        return;
    }
    const AcDesc d = desc[sidx];
    // kShared: the model lives in shared memory (LDS/STS, no generic accesses).
    // Capacity from the actual symbol count (the host sizes buffers from bounds).
    const u32 cap_need = static_cast<u32>(ns + 1);
    const u32 cap = kShared ? min(cap_need, smem_cap) : cap_need;
    u32* base = kShared ? reinterpret_cast<u32*>(ac_smem) : scratch + d.model_off;
    u32* cnt = base;
    u32* l1 = cnt + cap;
    u32* l2 = l1 + (cap / 32 + 1);
    u32* hidx = l2 + (cap / 1024 + 1);
    const u32 hb = log2_at_least(2 * cap);
    const u32 hmask = (1u << hb) - 1;
    u64* val = reinterpret_cast<u64*>(base + ((cap + (cap / 32 + 1) + (cap / 1024 + 1) + (1u << hb) + 1) & ~1u));
    for (u32 i = lane; i < cap; i += 32) cnt[i] = 0;
    for (u32 i = lane; i <= cap / 32; i += 32) l1[i] = 0;
    for (u32 i = lane; i <= cap / 1024; i += 32) l2[i] = 0;
    for (u32 i = lane; i < (1u << hb); i += 32) hidx[i] = 0;
    __syncwarp();
    u8* out = outbuf + d.out_off;
    if (lane == 0) {
        out[0] = 0;  // coder id: arithmetic
        const u32 cnt32 = static_cast<u32>(ns);
        for (int i = 0; i < 4; ++i) out[1 + i] = static_cast<u8>(cnt32 >> (8 * i));
        cnt[0] = 1;
        val[0] = 0;
        l1[0] = 1;
        l2[0] = 1;
    }
    __syncwarp();
    // range coder state (identical in every lane)
    u64 low = 0, pending = 1, pos = 5;
    u32 range = 0xFFFFFFFFu;
    u8 cache = 0;
    auto shift = [&]() {
        if (static_cast<u32>(low) < 0xFF000000u || (low >> 32) != 0) {
            // the cached byte and the pending 0xFF run (plus the carry), one byte per
            // lane: no serial loop, no divergent branch
            const u8 carry = static_cast<u8>(low >> 32);
            for (u64 q0 = 0; q0 < pending; q0 += 32) {
                const u64 q = q0 + static_cast<u64>(lane);
                if (q < pending) out[pos + q] = static_cast<u8>((q == 0 ? cache : u8{0xFF}) + carry);
            }
            pos += pending;
            pending = 0;
            cache = static_cast<u8>(low >> 24);
        }
        ++pending;
        low = (low << 8) & 0xFFFFFFFFull;
    };
    auto norm = [&]() {
        while (range < (1u << 24)) {
            shift();
            range <<= 8;
        }
    };
    u32 nsym = 1, total = 1;
    auto halve = [&]() {
        __syncwarp();
        for (u32 i = lane; i <= cap / 32; i += 32) l1[i] = 0;
        for (u32 i = lane; i <= cap / 1024; i += 32) l2[i] = 0;
        __syncwarp();
        u32 t = 0;
        for (u32 i0 = 0; i0 < nsym; i0 += 32) {
            const u32 i = i0 + lane;
            u32 c = 0;
            if (i < nsym) {
                c = max(1u, cnt[i] >> 1);
                cnt[i] = c;
            }
            u32 bs = c;  // block i0/32 sum
            for (int o = 16; o > 0; o >>= 1) bs += __shfl_xor_sync(0xffffffffu, bs, o);
            if (lane == 0) {
                l1[i0 >> 5] = bs;
                l2[i0 >> 10] += bs;
            }
            t += bs;
            __syncwarp();
        }
        total = t;
        __syncwarp();
    };
    // Chunked model: between halvings the adaptive model (entropy.cpp:155-239)
    // has a closed form, so 32 symbols (lane l <-> symbol t0 + l) resolve in
    // parallel against the model as of t0:
    //   index I: hash lookup, else a new symbol; repeats inside the chunk share
    //            the first occurrence's index (match_any), new indices follow
    //            first-occurrence order (ballot prefix);
    //   cum     = count below I at t0 + 32 * #{earlier chunk symbols with index < I};
    //   freq    = count of I at t0 + 32 * #{earlier chunk occurrences of I};
    //   total   = total(t0) + 32 l; escapes code (0, cnt[0] = 1, total).
    // A chunk ends at the first halving point (after coding the symbol whose
    // pre-update total + 32 reaches 2^16), applied between that symbol's
    // coding and its increment.  Only the range-coder arithmetic is sequential.
    const u64* sy = syms + d.sym_off;
    const unsigned below_me = (1u << lane) - 1u;
    u64 cur = lane < ns ? sy[lane] : 0;
    for (u64 t0 = 0; t0 < ns;) {
        u32 L = static_cast<u32>(ns - t0 < 32 ? ns - t0 : 32);
        // first l with total + 32 l + 32 >= 2^16 (total < 2^16 between symbols)
        const u32 lh = total >= 65504u ? 0u : (65504u - total + 31u) / 32u;
        const bool halv = lh < L;
        if (halv) L = lh + 1;
        const u64 nxt = t0 + L + lane < ns ? sy[t0 + L + lane] : 0;  // next chunk, in flight
        const bool act = static_cast<u32>(lane) < L;
        const u64 sv = cur;
        int I = -1;
        if (act) {
            u32 h = hslot(sv, hb);
            while (true) {
                const u32 e = hidx[h];
                if (e == 0) break;
                if (val[e - 1] == sv) {
                    I = static_cast<int>(e) - 1;
                    break;
                }
                h = (h + 1) & hmask;
            }
        }
        const unsigned am = __ballot_sync(0xffffffffu, act);
        const unsigned same = __match_any_sync(0xffffffffu, sv) & am;
        const int leader = act ? __ffs(same) - 1 : lane;
        const bool isnew = act && I < 0 && leader == lane;
        const unsigned newm = __ballot_sync(0xffffffffu, isnew);
        if (nsym + __popc(newm) > cap) {  // model full: rerun from global scratch
            if (lane == 0) {
                *redo = 1;
                elen[sidx] = ~u64{0};
            }
            return;
        }
        if (isnew) I = static_cast<int>(nsym + __popc(newm & below_me));
        const int IL = __shfl_sync(0xffffffffu, I, leader);
        if (act && I < 0) I = IL;
        u32 base = 0, f0 = 0;
        if (act) {
            const u32 ui = static_cast<u32>(I);
            if (ui < nsym) {
                const u32 b1 = ui >> 5, b2 = ui >> 10;
                for (u32 j = b1 << 5; j < ui; ++j) base += cnt[j];
                for (u32 j = b2 << 5; j < b1; ++j) base += l1[j];
                for (u32 j = 0; j < b2; ++j) base += l2[j];
                f0 = cnt[ui];
            } else {
                base = total;  // every index present at t0 is below a new one
            }
        }
        u32 within = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int Ij = __shfl_sync(0xffffffffu, I, j);
            within += (j < lane && Ij < I) ? 1u : 0u;
        }
        const u32 cum = isnew ? 0u : base + 32u * within;
        const u32 freq = isnew ? 1u : f0 + 32u * __popc(same & below_me);
        const u32 tot = total + 32u * static_cast<u32>(lane);
        // floor(range / T) by multiply-high: with m = ceil(2^64 / T) the product's high
        // word is exact for range < 2^32 and 1 < T < 2^32 (the error term is below
        // 2^-32 while a non-integer quotient is at least 1/T below the next integer);
        // each lane prepares its own T's multiplier off the sequential path.
        const u64 magic = tot > 1u ? (~u64{0} / tot) + 1u : 0u;
        // range coder over the chunk (identical state in every lane); symbol l + 1's
        // operands are fetched while symbol l is coded (the shuffles are off the
        // coder's dependency chain)
        u32 c = __shfl_sync(0xffffffffu, cum, 0), f = __shfl_sync(0xffffffffu, freq, 0);
        u32 T = __shfl_sync(0xffffffffu, tot, 0);
        u64 v = __shfl_sync(0xffffffffu, sv, 0), M = __shfl_sync(0xffffffffu, magic, 0);
        for (u32 l = 0; l < L; ++l) {
            const u32 ln = l + 1 < L ? l + 1 : l;
            const u32 c_n = __shfl_sync(0xffffffffu, cum, ln), f_n = __shfl_sync(0xffffffffu, freq, ln);
            const u32 T_n = __shfl_sync(0xffffffffu, tot, ln);
            const u64 v_n = __shfl_sync(0xffffffffu, sv, ln), M_n = __shfl_sync(0xffffffffu, magic, ln);
            range = T > 1u ? static_cast<u32>(__umul64hi(static_cast<u64>(range), M)) : range;
            low += static_cast<u64>(c) * range;
            range *= f;
            norm();
            if ((newm >> l) & 1u) {
                // 32 raw bits, MSB first, each encode(bit, 1, 2): range >>= 1; low += bit ?
                // range : 0; norm().  With range in [2^24, 2^32) exactly k = floor(log2
                // range) - 23 halvings happen before the next normalisation, so up to k
                // bits go at once: low += sum_j bit_j (range >> j), range >>= k, norm().
                // Identical arithmetic, about five groups instead of 32 steps.
                const u32 raw = static_cast<u32>(v);
                int left = 32;
                while (left > 0) {
                    const int k = min(left, (31 - __clz(static_cast<int>(range))) - 23);
                    const u32 cb = (raw >> (left - k)) & ((1u << k) - 1u);
                    u64 add = 0;
#pragma unroll
                    for (int j = 1; j <= 8; ++j)
                        if (j <= k && ((cb >> (k - j)) & 1u)) add += range >> j;
                    low += add;
                    range >>= k;
                    left -= k;
                    norm();
                }
            }
            c = c_n;
            f = f_n;
            T = T_n;
            v = v_n;
            M = M_n;
        }
        // model update: increments in symbol order, a halving before the last one
        auto inc = [&](bool doit) {
            if (!doit) return;
            const u32 ui = static_cast<u32>(I);
            if (isnew) {
                val[ui] = sv;
                u32 h = hslot(sv, hb);
                while (atomicCAS(&hidx[h], 0u, ui + 1u) != 0u) h = (h + 1) & hmask;
            }
            atomicAdd(&cnt[ui], 32u);
            atomicAdd(&l1[ui >> 5], 32u);
            atomicAdd(&l2[ui >> 10], 32u);
        };
        if (halv) {
            const unsigned lastbit = 1u << (L - 1);
            inc(act && static_cast<u32>(lane) != L - 1);
            nsym += __popc(newm & ~lastbit);
            halve();
            inc(static_cast<u32>(lane) == L - 1);
            nsym += (newm & lastbit) ? 1u : 0u;
            total += 32u;
        } else {
            inc(act);
            nsym += __popc(newm);
            total += 32u * L;
        }
        __syncwarp();
        t0 += L;
        cur = nxt;
    }
    for (int i = 0; i < 5; ++i) shift();
    if (lane == 0) elen[sidx] = pos;
}

// Host side: shared-memory pass for every stream, global-scratch rerun for
// the ones whose model overflowed.
void run_ac(const u64* syms, const StreamOut* so, const AcDesc* dad, const std::vector<AcDesc>& ad,
            const std::vector<StreamOut>& soh, int ns, u8* ent, u32* scratch, u64* elen, cudaStream_t s) {
    u32 need = 0;
    for (int i = 0; i < ns; ++i)
        if (soh[i].nsyms) need = std::max<u32>(need, std::min<u32>(ad[i].cap, kAcSmemCap));
    if (need == 0) {
        TCB_CUDA(cudaMemsetAsync(elen, 0, ns * sizeof(u64), s));
        return;
    }
    const u64 smem = ac_model_words(need) * 4 + 16;
    static bool attr = [] {
        cudaFuncSetAttribute(ac_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(ac_model_words(kAcSmemCap) * 4 + 16));
        return true;
    }();
    (void)attr;
    DevBuf<int> redo(1, s);
    redo.zero();
    {
        ProfScope pa(kAc, s);
        ac_kernel<true><<<static_cast<unsigned>(ns), 32, smem, s>>>(syms, so, dad, nullptr, ns, ent, scratch, elen, need,
                                                             redo.p);
    }
    count_launch();
    TCB_LAUNCH();
    if (redo.to_host()[0] == 0) return;
    std::vector<u64> el(ns);
    d2h(el.data(), elen, ns * sizeof(u64), s);
    stream_sync(s);
    std::vector<int> ids;
    for (int i = 0; i < ns; ++i)
        if (el[i] == ~u64{0}) ids.push_back(i);
    DevBuf<int> dids(ids.size(), s);
    dids.upload(ids.data(), ids.size());
    {
        ProfScope pa(kAc, s);
        ac_kernel<false><<<static_cast<unsigned>(ids.size()), 32, 0, s>>>(syms, so, dad, dids.p, ns, ent, scratch, elen, 0,
                                                                  redo.p);
    }
    count_launch();
    TCB_LAUNCH();
}

// Launch-only variant for emit_planes: every stream's shared-memory pass with
// the largest model that fits; streams whose model overflows report ~0 in
// elen and are rerun by the caller from global scratch once the lengths are
// back on the host (no extra round trip in the common case).
void launch_ac_shared(const u64* syms, const StreamOut* so, const AcDesc* dad, int ns, u8* ent, u64* elen,
                      int* redo, cudaStream_t s) {
    const u64 smem = ac_model_words(kAcSmemCap) * 4 + 16;
    static bool attr = [] {
        cudaFuncSetAttribute(ac_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(ac_model_words(kAcSmemCap) * 4 + 16));
        return true;
    }();
    (void)attr;
    ProfScope pa(kAc, s);
    ac_kernel<true><<<static_cast<unsigned>(ns), 32, smem, s>>>(syms, so, dad, nullptr, ns, ent, nullptr, elen,
                                                         kAcSmemCap, redo);
    count_launch();
    TCB_LAUNCH();
}

// ---------------------------------------------------------------- semi-static rANS (entropy.cpp:290-421)
// One warp per stream, lane 0: histogram through an open-addressing hash
// (first-occurrence indices), the distinct symbols heap-sorted by value, the
// reference's table normalisation (floor-scaled counts, then +-1 on the first
// largest count until the total is 2^bits, bits = max(12, ceil log2 distinct)),
// then the backwards encode; output framing as the range coder's (coder id 1,
// u32 count, varint table, 8-byte state, 32-bit words in reverse).
__host__ __device__ inline u64 rans_scratch_words(u64 nsyms) {
    const u64 cap = nsyms + 1;
    const u64 hs = u64{1} << log2_at_least(static_cast<u32>(2 * cap));
    return 2 * cap /*val*/ + 2 * cap /*cnt*/ + hs /*hash*/ + 4 * cap /*order,f,pos,c*/ + 4 + (nsyms + 4) /*words*/ + 2;
}
__host__ __device__ inline u64 rans_out_cap(u64 nsyms) { return 24 * nsyms + 64; }

__global__ void __launch_bounds__(32) rans_kernel(const u64* __restrict__ syms, const StreamOut* __restrict__ sout,
                                                  const AcDesc* __restrict__ desc, int nstreams, u8* __restrict__ outbuf,
                                                  u32* __restrict__ scratch, u64* __restrict__ elen) {
    const int sidx = static_cast<int>(blockIdx.x);
    if (sidx >= nstreams || threadIdx.x != 0) return;
    const u64 N = sout[sidx].nsyms;
    if (N == 0) {
        elen[sidx] = 0;
        return;
    }
    const AcDesc d = desc[sidx];
    const u64* sy = syms + d.sym_off;
    u8* out = outbuf + d.out_off;
    const u64 cap = N + 1;
    const u32 hb = log2_at_least(static_cast<u32>(2 * cap));
    const u32 hmask = (1u << hb) - 1;
    u32* base = scratch + d.model_off;  // 8-byte aligned by the host
    u64* val = reinterpret_cast<u64*>(base);
    u64* cnt = val + cap;
    u32* hidx = reinterpret_cast<u32*>(cnt + cap);
    u32* order = hidx + (1u << hb);
    u32* f = order + cap;
    u32* pos = f + cap;
    u32* c = pos + cap;
    u32* words = c + cap + 1;
    for (u32 i = 0; i <= hmask; ++i) hidx[i] = 0;
    u32 nd = 0;
    for (u64 t = 0; t < N; ++t) {  // histogram, first-occurrence indices
        const u64 s = sy[t];
        u32 h = hslot(s, hb);
        while (true) {
            const u32 e = hidx[h];
            if (e == 0) {
                val[nd] = s;
                cnt[nd] = 1;
                hidx[h] = ++nd;
                break;
            }
            if (val[e - 1] == s) {
                ++cnt[e - 1];
                break;
            }
            h = (h + 1) & hmask;
        }
    }
    // heap sort of the distinct indices by value
    for (u32 i = 0; i < nd; ++i) order[i] = i;
    auto sift = [&](u32 root, u32 end) {
        while (2 * root + 1 < end) {
            u32 ch = 2 * root + 1;
            if (ch + 1 < end && val[order[ch + 1]] > val[order[ch]]) ++ch;
            if (val[order[root]] >= val[order[ch]]) return;
            const u32 tmp = order[root];
            order[root] = order[ch];
            order[ch] = tmp;
            root = ch;
        }
    };
    for (u32 i = nd / 2; i-- > 0;) sift(i, nd);
    for (u32 end = nd; end-- > 1;) {
        const u32 tmp = order[0];
        order[0] = order[end];
        order[end] = tmp;
        sift(0, end);
    }
    u32 bits = 12;
    while ((u64{1} << bits) < nd) ++bits;
    const u64 scale = u64{1} << bits;
    u64 sum = 0;
    for (u32 j = 0; j < nd; ++j) {
        u64 q = cnt[order[j]] * scale / N;
        if (q == 0) q = 1;
        f[j] = static_cast<u32>(q);
        pos[order[j]] = j;
        sum += q;
    }
    while (sum != scale) {
        const bool grow = sum < scale;
        u32 pick = 0;
        for (u32 i = 1; i < nd; ++i) {
            const bool better = grow ? f[i] > f[pick] : (f[i] > f[pick] && f[i] > 1);
            if (better) pick = i;
        }
        if (grow) {
            ++f[pick];
            ++sum;
        } else {
            if (f[pick] <= 1) {  // the reference throws "entropy: cannot normalize rans table"
                elen[sidx] = ~u64{1};
                return;
            }
            --f[pick];
            --sum;
        }
    }
    c[0] = 0;
    for (u32 j = 0; j < nd; ++j) c[j + 1] = c[j] + f[j];
    // header: coder id, u32 count, varint table
    u64 o = 0;
    out[o++] = 1;
    for (int i = 0; i < 4; ++i) out[o++] = static_cast<u8>(static_cast<u32>(N) >> (8 * i));
    auto varint = [&](u64 v) {
        for (; v >= 0x80; v >>= 7) out[o++] = static_cast<u8>(v) | 0x80u;
        out[o++] = static_cast<u8>(v);
    };
    varint(nd);
    varint(bits);
    u64 prev = 0;
    for (u32 j = 0; j < nd; ++j) {
        varint(val[order[j]] - prev);
        varint(f[j]);
        prev = val[order[j]];
    }
    // backwards encode
    constexpr u64 L = u64{1} << 31;
    u64 x = L;
    u64 nw = 0;
    for (u64 t = N; t-- > 0;) {
        const u64 s = sy[t];
        u32 h = hslot(s, hb);
        while (val[hidx[h] - 1] != s) h = (h + 1) & hmask;
        const u32 j = pos[hidx[h] - 1];
        const u64 fj = f[j];
        const u64 lim = ((L >> bits) << 32) * fj;
        while (x >= lim) {
            words[nw++] = static_cast<u32>(x);
            x >>= 32;
        }
        x = ((x / fj) << bits) + (x % fj) + c[j];
    }
    for (int i = 0; i < 8; ++i) out[o++] = static_cast<u8>(x >> (8 * i));
    for (u64 w = nw; w-- > 0;)
        for (int b = 0; b < 4; ++b) out[o++] = static_cast<u8>(words[w] >> (8 * b));
    elen[sidx] = o;
}

void run_rans(const u64* syms, const StreamOut* so, const AcDesc* dad, int ns, u8* ent, u32* scratch, u64* elen,
              cudaStream_t s) {
    if (ns == 0) return;
    {
        ProfScope pa(kAc, s);
        rans_kernel<<<static_cast<unsigned>(ns), 32, 0, s>>>(syms, so, dad, ns, ent, scratch, elen);
    }
    count_launch();
    TCB_LAUNCH();
}

// ---------------------------------------------------------------- assembly
__global__ void assemble_kernel(const u8* __restrict__ ent, const AcDesc* __restrict__ acd,
                                const u64* __restrict__ elen, const u32* __restrict__ raw,
                                const StreamDesc* __restrict__ sd, const StreamOut* __restrict__ so,
                                const u64* __restrict__ dst_off, u8* __restrict__ body) {
    const int s = blockIdx.x;
    const u64 el = elen[s];
    const u64 rb = (so[s].nraw + 7) / 8;
    const u64 payload = 4 + el + rb;
    u8* o = body + dst_off[s];
    if (threadIdx.x < 4) {
        o[threadIdx.x] = static_cast<u8>(static_cast<u32>(payload) >> (8 * threadIdx.x));
        o[4 + threadIdx.x] = static_cast<u8>(static_cast<u32>(el) >> (8 * threadIdx.x));
    }
    const u8* e = ent + acd[s].out_off;
    for (u64 i = threadIdx.x; i < el; i += blockDim.x) o[8 + i] = e[i];
    const u64 rbyte0 = sd[s].raw_off >> 3;
    const u8* rbytes = reinterpret_cast<const u8*>(raw);
    for (u64 i = threadIdx.x; i < rb; i += blockDim.x) o[8 + el + i] = rbytes[rbyte0 + i];
}

}  // namespace

// ================================================================ host launchers
SumRec device_sum(SumKind kind, const u64* m, const u64* dec, u64 n, int plane, cudaStream_t s) {
    ProfScope prof_scope(kSum, s);
    const int grid = grid_for(n, kSumThreads, 4, 4);
    DevBuf<SumRec> part(grid, s);
    sum_kernel<<<grid, kSumThreads, 0, s>>>(kind, m, dec, n, plane, part.p);
    count_launch();
    TCB_LAUNCH();
    auto h = part.to_host();
    // fixed-order double-double combine on the host
    double hi = 0.0, lo = 0.0, w = 0.0;
    for (const auto& r : h) {
        const double s1 = hi + r.hi;
        const double bb = s1 - hi;
        const double e1 = (hi - (s1 - bb)) + (r.hi - bb);
        const double e = e1 + lo + r.lo;
        hi = s1 + e;
        lo = e - (hi - s1);
        w += r.wabs;
    }
    return SumRec{hi, lo, w, n};
}

double device_sum_serial(SumKind kind, const u64* m, const u64* dec, u64 n, int plane, cudaStream_t s) {
    ProfScope prof_scope(kSum, s);
    DevBuf<double> out(1, s);
    sum_serial_kernel<<<1, kSerThreads, 0, s>>>(kind, m, dec, n, plane, out.p);
    count_launch();
    TCB_LAUNCH();
    return out.to_host()[0];
}

void plane_stats(const u64* m, u64 n, u64 block, int p_hi, int p_lo, PlaneBlockRec* out_host, cudaStream_t s) {
    ProfScope prof_scope(kStats, s);
    const u64 nb = (n + block - 1) / block;
    const u64 cpb = (block + kChunk - 1) / kChunk;
    const int np = p_hi - p_lo + 1;
    DevBuf<Partial> part(nb * cpb * np, s);
    DevBuf<PlaneBlockRec> out(nb * np, s);
    dim3 grid(static_cast<unsigned>(nb * cpb), static_cast<unsigned>(np));
    stats_kernel<<<grid, kStatThreads, 0, s>>>(m, n, block, cpb, p_hi, part.p);
    stats_combine<<<cdiv(nb * np, 128), 128, 0, s>>>(part.p, nb, cpb, np, out.p, n, block);
    count_launch(2);
    TCB_LAUNCH();
    out.download(out_host, nb * np);
    stream_sync(s);
}

void plane_stats_serial(const u64* m, u64 n, u64 block, int p, PlaneBlockRec* out_host, cudaStream_t s) {
    ProfScope prof_scope(kStats, s);
    const u64 nb = (n + block - 1) / block;
    DevBuf<PlaneBlockRec> out(nb, s);
    stats_serial_kernel<<<dim3(static_cast<unsigned>(nb), 1), kSerThreads, 0, s>>>(m, n, block, nb, p, out.p);
    count_launch();
    TCB_LAUNCH();
    out.download(out_host, nb);
    stream_sync(s);
}

std::vector<double> device_sums_serial(const std::vector<std::pair<SumKind, int>>& list, const u64* m, u64 n,
                                       cudaStream_t s) {
    ProfScope prof_scope(kSum, s);
    const int k = static_cast<int>(list.size());
    if (k == 0) return {};
    std::vector<int> kinds(k), planes(k);
    for (int i = 0; i < k; ++i) {
        kinds[i] = static_cast<int>(list[i].first);
        planes[i] = list[i].second;
    }
    DevBuf<int> dk(k, s), dp(k, s);
    dk.upload(kinds.data(), k);
    dp.upload(planes.data(), k);
    DevBuf<double> out(k, s);
    sum_serial_multi_kernel<<<static_cast<unsigned>(k), kSerThreads, 0, s>>>(dk.p, dp.p, m, n, out.p);
    count_launch();
    TCB_LAUNCH();
    return out.to_host();
}

void plane_stats_serial_range(const u64* m, u64 n, u64 block, int p_hi, int p_lo, PlaneBlockRec* out_host,
                              cudaStream_t s) {
    ProfScope prof_scope(kStats, s);
    const u64 nb = (n + block - 1) / block;
    const int np = p_hi - p_lo + 1;
    DevBuf<PlaneBlockRec> out(nb * np, s);
    stats_serial_kernel<<<dim3(static_cast<unsigned>(nb), static_cast<unsigned>(np)), kSerThreads, 0, s>>>(
        m, n, block, nb, p_hi, out.p);
    count_launch();
    TCB_LAUNCH();
    out.download(out_host, nb * np);
    stream_sync(s);
}

void crossing_scan(const u64* m, u64 n, u64 block, u64 b, int plane, int category, const double* cum,
                   const double* need, int npairs, u64* counts_host, cudaStream_t s) {
    ProfScope prof_scope(kStats, s);
    DevBuf<double> c(npairs, s), nd(npairs, s);
    DevBuf<u64> out(2 * npairs, s);
    c.upload(cum, npairs);
    nd.upload(need, npairs);
    const u64 lo = b * block, hi = std::min<u64>(n, lo + block);
    if (npairs > kCrossThreads) throw Error("crossing scan: too many pairs");
    crossing_kernel<<<1, kCrossThreads, 0, s>>>(m, lo, hi, plane, category, c.p, nd.p, npairs, out.p);
    count_launch();
    TCB_LAUNCH();
    out.download(counts_host, 2 * npairs);
    stream_sync(s);
}

void decode_model(const u64* m, u64 n, u64 block, int last_plane, const u64* stops_dev, u64* dec, cudaStream_t s) {
    ProfScope prof_scope(kStats, s);
    const u64 nb = (n + block - 1) / block;
    if (nb == 0) return;
    decode_model_kernel<<<static_cast<unsigned>(nb), kDecThreads, 0, s>>>(m, n, block, last_plane, stops_dev, dec);
    count_launch();
    TCB_LAUNCH();
}

std::vector<u8> encode_symbols_device(int coder, const u64* syms_host, u64 n, cudaStream_t s) {
    if (coder != 0 && coder != 1) throw Error("entropy: unknown coder");
    if (coder == 1 && n > 0) {
        DevBuf<u64> syms(n, s);
        syms.upload(syms_host, n);
        StreamOut so{n, 0};
        DevBuf<StreamOut> dso(1, s);
        dso.upload(&so, 1);
        AcDesc a{};
        DevBuf<AcDesc> dad(1, s);
        dad.upload(&a, 1);
        DevBuf<u8> ent(rans_out_cap(n), s);
        DevBuf<u32> scratch(rans_scratch_words(n) + 2, s);
        DevBuf<u64> elen(1, s);
        run_rans(syms.p, dso.p, dad.p, 1, ent.p, scratch.p, elen.p, s);
        const u64 el = elen.to_host()[0];
        if (el == ~u64{1}) throw Error("entropy: cannot normalize rans table");
        std::vector<u8> out(el);
        ent.download(out.data(), el);
        stream_sync(s);
        return out;
    }
    std::vector<u8> out{static_cast<u8>(coder)};
    for (int i = 0; i < 4; ++i) out.push_back(static_cast<u8>(static_cast<u32>(n) >> (8 * i)));
    if (n == 0) return out;
    DevBuf<u64> syms(n, s);
    syms.upload(syms_host, n);
    StreamOut so{n, 0};
    DevBuf<StreamOut> dso(1, s);
    dso.upload(&so, 1);
    AcDesc a{};
    a.cap = static_cast<u32>(n + 1);
    a.hbits = log2_at_least(2 * a.cap);
    DevBuf<AcDesc> dad(1, s);
    dad.upload(&a, 1);
    DevBuf<u8> ent(5 + 7 * n + 16, s);
    DevBuf<u32> scratch(ac_model_words(a.cap) + 2, s);
    DevBuf<u64> elen(1, s);
    run_ac(syms.p, dso.p, dad.p, std::vector<AcDesc>{a}, std::vector<StreamOut>{so}, 1, ent.p, scratch.p, elen.p, s);
    const u64 el = elen.to_host()[0];
    out.resize(el);
    ent.download(out.data(), el);
    stream_sync(s);
    return out;
}

struct ProbeCache {
    u64 n = 0, nb = 0;
    int coder = 0;
    cudaStream_t s = nullptr;
    std::vector<StreamDesc> sd;
    std::vector<AcDesc> ad;
    DevBuf<StreamDesc> dsd;
    DevBuf<u64> syms;
    DevBuf<u32> raw;
    DevBuf<StreamOut> so;
    DevBuf<AcDesc> dad;
    DevBuf<u8> ent;
    DevBuf<u64> elen;
    DevBuf<u32> scratch;
    DevBuf<int> redo;
    cudaEvent_t done = nullptr;
    bool ready = false;
    std::vector<u64> el;
    std::mutex mu;
    ~ProbeCache() {
        if (done) {
            cudaEventSynchronize(done);
            cudaEventDestroy(done);
        }
    }
};

std::shared_ptr<ProbeCache> probe_planes_async(const u64* m, u64 n, u64 block, int coder, cudaStream_t side) {
    auto c = std::make_shared<ProbeCache>();
    c->n = n;
    c->coder = coder;
    c->s = side;
    const u64 nb = n == 0 ? 0 : (n + block - 1) / block;
    c->nb = nb;
    const u64 ns = nb * 64;
    if (ns == 0) return c;
    c->sd.resize(ns);
    u64 sym_total = 0, raw_words = 0;
    for (int pi = 0; pi < 64; ++pi)
        for (u64 b = 0; b < nb; ++b) {
            StreamDesc& d = c->sd[pi * nb + b];
            d.lo = b * block;
            d.hi = std::min<u64>(n, d.lo + block);
            d.plane = 63 - pi;
            d.lstop = d.tstop = kFull;
            d.sym_off = sym_total;
            sym_total += d.hi - d.lo + 1;
            d.raw_off = raw_words * 32;
            raw_words += (d.hi - d.lo + 31) / 32;
        }
    c->ad.resize(ns);
    u64 out_total = 0, scratch_total = 0;
    for (u64 i = 0; i < ns; ++i) {
        AcDesc& a = c->ad[i];
        const u64 kmax = c->sd[i].hi - c->sd[i].lo + 1;
        a.sym_off = c->sd[i].sym_off;
        a.out_off = out_total;
        a.cap = static_cast<u32>(kmax + 1);
        a.fen = 0;
        a.hbits = log2_at_least(2 * a.cap);
        if (coder == 1) {
            out_total += rans_out_cap(kmax);
            a.model_off = (scratch_total + 1) & ~u64{1};
            scratch_total = a.model_off + rans_scratch_words(kmax);
        } else {
            out_total += 5 + 7 * kmax + 16;
            a.model_off = 0;
        }
    }
    c->dsd = DevBuf<StreamDesc>(ns, side);
    c->dsd.upload(c->sd.data(), ns);
    c->syms = DevBuf<u64>(sym_total, side);
    c->raw = DevBuf<u32>(raw_words + 1, side);
    c->raw.zero();
    c->so = DevBuf<StreamOut>(ns, side);
    emit_kernel<<<static_cast<unsigned>(ns), kEmT, 0, side>>>(m, nullptr, c->dsd.p, c->syms.p, c->raw.p, c->so.p);
    count_launch();
    TCB_LAUNCH();
    c->dad = DevBuf<AcDesc>(ns, side);
    c->dad.upload(c->ad.data(), ns);
    c->ent = DevBuf<u8>(out_total + 1, side);
    c->elen = DevBuf<u64>(ns, side);
    c->scratch = DevBuf<u32>(coder == 1 ? scratch_total + 2 : 2, side);
    c->redo = DevBuf<int>(1, side);
    if (coder == 1) {
        run_rans(c->syms.p, c->so.p, c->dad.p, static_cast<int>(ns), c->ent.p, c->scratch.p, c->elen.p, side);
    } else {
        c->redo.zero();
        launch_ac_shared(c->syms.p, c->so.p, c->dad.p, static_cast<int>(ns), c->ent.p, c->elen.p, c->redo.p, side);
    }
    TCB_CUDA(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
    TCB_CUDA(cudaEventRecord(c->done, side));
    return c;
}

std::vector<u64> probe_entropy_bytes(ProbeCache& c, int p) {
    std::lock_guard<std::mutex> lk(c.mu);
    const u64 ns = c.nb * 64;
    if (!c.ready && ns > 0) {
        TCB_CUDA(cudaEventSynchronize(c.done));
        c.el.resize(ns);
        std::vector<StreamOut> soh(ns);
        c.elen.download(c.el.data(), ns);
        c.so.download(soh.data(), ns);
        stream_sync(c.s);
        if (c.coder == 0) {  // model overflow: rerun those streams from global scratch
            std::vector<int> ids;
            u64 words = 0;
            for (u64 i = 0; i < ns; ++i)
                if (c.el[i] == ~u64{0}) {
                    ids.push_back(static_cast<int>(i));
                    c.ad[i].model_off = words;
                    words += ac_model_words(static_cast<u32>(soh[i].nsyms + 1));
                }
            if (!ids.empty()) {
                DevBuf<u32> gscr(words + 2, c.s);
                c.dad.upload(c.ad.data(), ns);
                DevBuf<int> dids(ids.size(), c.s);
                dids.upload(ids.data(), ids.size());
                ac_kernel<false><<<static_cast<unsigned>(ids.size()), 32, 0, c.s>>>(
                    c.syms.p, c.so.p, c.dad.p, dids.p, static_cast<int>(ns), c.ent.p, gscr.p, c.elen.p, 0, c.redo.p);
                count_launch();
                TCB_LAUNCH();
                c.elen.download(c.el.data(), ns);
                stream_sync(c.s);
            }
        }
        for (u64 v : c.el)
            if (v == ~u64{1}) throw Error("entropy: cannot normalize rans table");
        c.ready = true;
    }
    std::vector<u64> out(c.nb);
    for (u64 b = 0; b < c.nb; ++b) out[b] = c.el[static_cast<u64>(63 - p) * c.nb + b];
    return out;
}

EmitResult emit_planes(const u64* m, const u8* neg, u64 n, u64 block, int last_plane, int top_plane,
                       const u64* stops_host, int coder, bool want_body, cudaStream_t s) {
    EmitResult res;
    if (coder != 0 && coder != 1) throw Error("entropy: unknown coder");
    const u64 nb = n == 0 ? 0 : (n + block - 1) / block;
    const int np = top_plane - last_plane + 1;
    const u64 ns = nb * static_cast<u64>(np);
    if (ns == 0 || np <= 0) return res;
    // upper bounds per stream: symbols <= positions + 1, raw bits <= positions
    std::vector<StreamDesc> sd(ns);
    u64 sym_total = 0, raw_words = 0;
    for (int pi = 0; pi < np; ++pi) {
        const int p = top_plane - pi;
        for (u64 b = 0; b < nb; ++b) {
            StreamDesc& d = sd[pi * nb + b];
            d.lo = b * block;
            d.hi = std::min<u64>(n, d.lo + block);
            d.plane = p;
            const bool bp = p == last_plane && stops_host != nullptr;
            d.lstop = bp ? stops_host[2 * b] : kFull;
            d.tstop = bp ? stops_host[2 * b + 1] : kFull;
            d.sym_off = sym_total;
            sym_total += d.hi - d.lo + 1;
            d.raw_off = raw_words * 32;
            raw_words += (d.hi - d.lo + 31) / 32;
        }
    }
    // No round trip between the symbol pass and the coder: entropy buffers are
    // sized from per-stream bounds (symbols <= positions + 1); the coder reads
    // the actual counts on the device.
    HostTrace ht_a("emit: symbols+entropy+sync");
    DevBuf<StreamDesc> dsd(ns, s);
    dsd.upload(sd.data(), ns);
    DevBuf<u64> syms(sym_total, s);
    DevBuf<u32> raw(raw_words + 1, s);
    raw.zero();
    DevBuf<StreamOut> so(ns, s);
    {
    ProfScope pe(kEmit, s);
    emit_kernel<<<static_cast<unsigned>(ns), kEmT, 0, s>>>(m, neg, dsd.p, syms.p, raw.p, so.p);
    }
    count_launch();
    TCB_LAUNCH();
    std::vector<AcDesc> ad(ns);
    u64 out_total = 0, scratch_total = 0;
    for (u64 i = 0; i < ns; ++i) {
        AcDesc& a = ad[i];
        a.sym_off = sd[i].sym_off;
        const u64 kmax = sd[i].hi - sd[i].lo + 1;
        a.out_off = out_total;
        a.cap = static_cast<u32>(kmax + 1);
        a.fen = 0;
        a.hbits = log2_at_least(2 * a.cap);
        if (coder == 1) {
            out_total += rans_out_cap(kmax);
            a.model_off = (scratch_total + 1) & ~u64{1};
            scratch_total = a.model_off + rans_scratch_words(kmax);
        } else {
            out_total += 5 + 7 * kmax + 16;
            a.model_off = 0;  // global scratch only for an overflow rerun (set below)
        }
    }
    DevBuf<AcDesc> dad(ns, s);
    dad.upload(ad.data(), ns);
    DevBuf<u8> ent(out_total + 1, s);
    DevBuf<u64> elen(ns, s);
    DevBuf<u32> scratch(coder == 1 ? scratch_total + 2 : 2, s);
    DevBuf<int> redo(1, s);
    if (coder == 1) {
        run_rans(syms.p, so.p, dad.p, static_cast<int>(ns), ent.p, scratch.p, elen.p, s);
    } else {
        redo.zero();
        launch_ac_shared(syms.p, so.p, dad.p, static_cast<int>(ns), ent.p, elen.p, redo.p, s);
    }
    std::vector<u64> el(ns);
    std::vector<StreamOut> soh(ns);
    elen.download(el.data(), ns);
    so.download(soh.data(), ns);
    stream_sync(s);
    if (coder == 0) {  // rerun the streams whose model outgrew shared memory from global scratch
        std::vector<int> ids;
        u64 words = 0;
        for (u64 i = 0; i < ns; ++i)
            if (el[i] == ~u64{0}) {
                ids.push_back(static_cast<int>(i));
                ad[i].model_off = words;
                words += ac_model_words(static_cast<u32>(soh[i].nsyms + 1));
            }
        if (!ids.empty()) {
            DevBuf<u32> gscr(words + 2, s);
            dad.upload(ad.data(), ns);
            DevBuf<int> dids(ids.size(), s);
            dids.upload(ids.data(), ids.size());
            {
                ProfScope pa(kAc, s);
                ac_kernel<false><<<static_cast<unsigned>(ids.size()), 32, 0, s>>>(
                    syms.p, so.p, dad.p, dids.p, static_cast<int>(ns), ent.p, gscr.p, elen.p, 0, redo.p);
            }
            count_launch();
            TCB_LAUNCH();
            elen.download(el.data(), ns);
            stream_sync(s);
        }
    }
    for (u64 v : el)
        if (v == ~u64{1}) throw Error("entropy: cannot normalize rans table");
    res.entropy_bytes = el;
    ht_a.stop();
    if (!want_body) return res;
    HostTrace ht_b("emit: assemble+sync");
    std::vector<u64> off(ns);
    u64 tot = 0;
    for (u64 i = 0; i < ns; ++i) {
        off[i] = tot;
        tot += 4 + 4 + el[i] + (soh[i].nraw + 7) / 8;
    }
    DevBuf<u64> doff(ns, s);
    doff.upload(off.data(), ns);
    DevBuf<u8> body(tot, s);
    ProfScope pz(kEmit, s);
    assemble_kernel<<<static_cast<unsigned>(ns), 128, 0, s>>>(ent.p, dad.p, elen.p, raw.p, dsd.p, so.p, doff.p,
                                                               body.p);
    count_launch();
    TCB_LAUNCH();
    res.body.resize(tot);
    body.download(res.body.data(), tot);
    stream_sync(s);
    return res;
}

}  // namespace tcb
