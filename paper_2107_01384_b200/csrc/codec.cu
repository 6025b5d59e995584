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
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <cfloat>

#include "ac.cuh"
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

// In 8192-position sub-chunks (all at once): lead / trail counts per sub-chunk,
// their prefix per block, then every position's decoded magnitude with the
// block's stops (the lead / trail index of a position is its sub-chunk's prefix
// plus a CTA scan).
constexpr u64 kDmSc = static_cast<u64>(kDecThreads) * 32;

__global__ void __launch_bounds__(kDecThreads) dm_count_kernel(const u64* __restrict__ m, u64 n, u64 block, u64 spb,
                                                                int lp, unsigned long long* __restrict__ cnt) {
    __shared__ unsigned long long sh[2];
    const u64 b = blockIdx.x / spb, j = blockIdx.x % spb;
    const u64 lo = b * block + j * kDmSc, hi = min(min(n, (b + 1) * block), lo + kDmSc);
    if (threadIdx.x < 2) sh[threadIdx.x] = 0;
    __syncthreads();
    u32 nl = 0, nt = 0;
    for (u64 i = lo + threadIdx.x; i < hi; i += kDecThreads) {
        const int t = top_bit(m[i]);
        nl += t <= lp;
        nt += t > lp;
    }
    for (int o = 16; o > 0; o >>= 1) {
        nl += __shfl_xor_sync(0xffffffffu, nl, o);
        nt += __shfl_xor_sync(0xffffffffu, nt, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&sh[0], static_cast<unsigned long long>(nl));
        atomicAdd(&sh[1], static_cast<unsigned long long>(nt));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        cnt[2 * blockIdx.x] = sh[0];
        cnt[2 * blockIdx.x + 1] = sh[1];
    }
}

__global__ void dm_scan_kernel(unsigned long long* __restrict__ cnt, u64 nb, u64 spb) {
    const u64 b = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    unsigned long long L = 0, T = 0;
    for (u64 j = 0; j < spb; ++j) {
        unsigned long long* c = cnt + 2 * (b * spb + j);
        const unsigned long long l = c[0], t = c[1];
        c[0] = L;
        c[1] = T;
        L += l;
        T += t;
    }
}

// Warp w of the CTA owns positions [lo + 1024 w, lo + 1024 (w + 1)) as rows of
// 32: a position's lead / trail index is the sub-chunk prefix, the counts of
// the warps before it and a popcount of its row's ballot (coalesced rows).
__global__ void __launch_bounds__(kDecThreads) dm_decode_kernel(const u64* __restrict__ m, u64 n, u64 block, u64 spb,
                                                                 int lp, const u64* __restrict__ stops,
                                                                 const unsigned long long* __restrict__ cnt,
                                                                 u64* __restrict__ dec) {
    __shared__ u32 wc[kDecThreads / 32][2];
    const u64 b = blockIdx.x / spb, j = blockIdx.x % spb;
    const u64 lo = b * block + j * kDmSc, hi = min(min(n, (b + 1) * block), lo + kDmSc);
    const u64 lstop = stops[2 * b], tstop = stops[2 * b + 1];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const u64 wlo = lo + static_cast<u64>(w) * 1024;
    u32 nl = 0, nt = 0;
    for (int r = 0; r < 32; ++r) {
        const u64 i = wlo + static_cast<u64>(r) * 32 + lane;
        const int t = i < hi ? top_bit(m[i]) : 1000;
        nl += __popc(__ballot_sync(0xffffffffu, t <= lp));
        nt += __popc(__ballot_sync(0xffffffffu, t > lp && t < 1000));
    }
    if (lane == 0) {
        wc[w][0] = nl;
        wc[w][1] = nt;
    }
    __syncthreads();
    u64 li = cnt[2 * blockIdx.x], ti = cnt[2 * blockIdx.x + 1];
    for (int q = 0; q < w; ++q) {
        li += wc[q][0];
        ti += wc[q][1];
    }
    for (int r = 0; r < 32; ++r) {
        const u64 i = wlo + static_cast<u64>(r) * 32 + lane;
        const u64 v = i < hi ? m[i] : 0;
        const int t = i < hi ? top_bit(v) : 1000;
        const unsigned lm = __ballot_sync(0xffffffffu, t <= lp), tm = __ballot_sync(0xffffffffu, t > lp && t < 1000);
        int pe = -1;
        if (t > lp && t < 1000) {
            pe = (ti + __popc(tm & lt) < tstop) ? lp : lp + 1;
        } else if (t == lp && li + __popc(lm & lt) < lstop) {
            pe = lp;
        }
        u64 out = 0;
        if (pe >= 0) {
            out = pe >= 64 ? 0 : (v >> pe) << pe;
            if (pe >= 1 && pe < 64) out += u64{1} << (pe - 1);
        }
        if (i < hi) dec[i] = out;
        li += __popc(lm);
        ti += __popc(tm);
    }
}

// ---------------------------------------------------------------- emission

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

// ---------------------------------------------------------------- parallel emission
// Every (plane, block) stream at once, in 8192-position sub-chunks: the
// sub-chunks' msb histograms give each stream's lead / trail / one counts
// before any sub-chunk (only a breakpoint stream's lead-stop crossing needs a
// scan), so one CTA per sub-chunk emits every plane from register-resident
// magnitudes: CTA scans place the symbols and raw bits; a sub-chunk's first
// zero-run symbol (which needs the previous sub-chunk's last one) is fixed up
// per stream afterwards.
constexpr int kScT = 256, kScPer = 32;
constexpr u64 kSc = static_cast<u64>(kScT) * kScPer;

struct ScOff {
    u64 lead_b, trail_b, ones_b, raw_b;  // positions / symbols / raw bits before the sub-chunk
};

__device__ __forceinline__ int sc_block(const u64* __restrict__ scoff, int nb, u64 g) {
    int lo = 0, hi = nb - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (scoff[mid] <= g) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(kScT) sc_hist_kernel(const u64* __restrict__ m, const StreamDesc* __restrict__ sd,
                                                       const u64* __restrict__ scoff, int nb, u32* __restrict__ hist) {
    __shared__ u32 h[65];
    const u64 g = blockIdx.x;
    const int bi = sc_block(scoff, nb, g);
    const StreamDesc d = sd[bi];  // plane-major layout: stream bi is block bi of the top plane
    const u64 lo = d.lo + (g - scoff[bi]) * kSc, hi = min(d.hi, lo + kSc);
    for (int i = threadIdx.x; i < 65; i += kScT) h[i] = 0;
    __syncthreads();
    for (u64 i0 = lo; i0 < hi; i0 += kScT) {
        const u64 i = i0 + threadIdx.x;
        const int bin = i < hi ? top_bit(m[i]) + 1 : -1;
        const unsigned act = __ballot_sync(0xffffffffu, bin >= 0);
        const unsigned same = __match_any_sync(0xffffffffu, bin) & act;
        if (bin >= 0 && (__ffs(same) - 1) == static_cast<int>(threadIdx.x & 31)) atomicAdd(&h[bin], __popc(same));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 65; i += kScT) hist[g * 65 + i] = h[i];
}

// One warp per stream: the offsets of every sub-chunk, and the stream's sizes.
// Lane l takes a contiguous range of the stream's sub-chunks; the lead / trail
// / one counts come from the sub-chunk msb histograms, prefixes by warp scans;
// only the sub-chunk where the lead stop falls (a breakpoint plane) is scanned
// element by element, by the lane that owns it.
__device__ __forceinline__ u64 warp_excl_scan_u64(u64 v, u64& total) {
    const int lane = threadIdx.x & 31;
    u64 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u64 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

__global__ void __launch_bounds__(128) sc_scan_kernel(const u64* __restrict__ m, const StreamDesc* __restrict__ sd,
                                                      int ns, int nb, const u64* __restrict__ scoff, u64 nsc_all,
                                                      const u32* __restrict__ hist, ScOff* __restrict__ tab,
                                                      StreamOut* __restrict__ so, u64* __restrict__ ncol_out) {
    const int st = static_cast<int>((static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    if (st >= ns) return;
    const int lane = threadIdx.x & 31;
    const StreamDesc d = sd[st];
    const int bi = st % nb, pi = st / nb, p = d.plane;
    const u64 nsc = scoff[bi + 1] - scoff[bi];
    ScOff* tb = tab + static_cast<u64>(pi) * nsc_all + scoff[bi];
    const u32* hb = hist + scoff[bi] * 65;
    const u64 per = (nsc + 31) / 32, j0 = min(nsc, lane * per), j1 = min(nsc, j0 + per);
    auto counts = [&](u64 j, u64& lead, u64& trail, u64& ones) {
        const u32* h = hb + j * 65;
        lead = 0;
        trail = 0;
        for (int q = 0; q <= p + 1; ++q) lead += h[q];
        for (int q = p + 2; q < 65; ++q) trail += h[q];
        ones = h[p + 1];
    };
    // pass 1: lead / trail totals of this lane's range, their prefixes
    u64 Ll = 0, Tl = 0;
    for (u64 j = j0; j < j1; ++j) {
        u64 l, t, o;
        counts(j, l, t, o);
        Ll += l;
        Tl += t;
    }
    u64 LT, TT;
    const u64 LB0 = warp_excl_scan_u64(Ll, LT), TB0 = warp_excl_scan_u64(Tl, TT);
    // the sub-chunk where the lead stop falls (LB + lead > lstop), if any
    u64 jc = ~u64{0};
    {
        u64 LB = LB0;
        for (u64 j = j0; j < j1 && jc == ~u64{0}; ++j) {
            u64 l, t, o;
            counts(j, l, t, o);
            if (LB + l > d.lstop) jc = j;
            LB += l;
        }
    }
    const unsigned has = __ballot_sync(0xffffffffu, jc != ~u64{0});
    const int owner = has ? __ffs(has) - 1 : -1;
    jc = owner >= 0 ? __shfl_sync(0xffffffffu, jc, owner) : ~u64{0};
    u64 part = 0;  // the crossing sub-chunk's ones up to the stop
    if (lane == owner) {
        u64 li = LB0;
        for (u64 j = j0; j < jc; ++j) {
            u64 l, t, o;
            counts(j, l, t, o);
            li += l;
        }
        const u64 lo = d.lo + jc * kSc, hi = min(d.hi, lo + kSc);
        for (u64 i = lo; i < hi && li < d.lstop; ++i) {
            const int t = top_bit(m[i]);
            if (t <= p) {
                part += t == p;
                ++li;
            }
        }
    }
    part = owner >= 0 ? __shfl_sync(0xffffffffu, part, owner) : 0;
    // pass 2: ones before each sub-chunk (all of them before the crossing, `part` at it)
    u64 Ol = 0;
    for (u64 j = j0; j < j1; ++j) {
        u64 l, t, o;
        counts(j, l, t, o);
        Ol += j < jc ? o : (j == jc ? part : 0);
    }
    u64 OT;
    const u64 OB0 = warp_excl_scan_u64(Ol, OT);
    // pass 3: the table
    u64 LB = LB0, TB = TB0, OB = OB0;
    for (u64 j = j0; j < j1; ++j) {
        u64 l, t, o;
        counts(j, l, t, o);
        tb[j] = ScOff{LB, TB, OB, min(TB, d.tstop) + OB};
        LB += l;
        TB += t;
        OB += j < jc ? o : (j == jc ? part : 0);
    }
    if (lane == 0) {
        const u64 ncol = min(LT, d.lstop);
        so[st] = StreamOut{ncol > 0 ? OT + 1 : 0, min(TT, d.tstop) + OT};
        ncol_out[st] = ncol;
    }
}

// One CTA per sub-chunk, every plane of the layout.  Warp w owns positions
// [lo + 1024 w, lo + 1024 (w + 1)) as 32 rows of 32 (row r, lane l: position
// lo + 1024 w + 32 r + l): loads and stores are coalesced, and a position's
// index among the lead / trail / one / raw positions of its row is a popcount
// of a ballot.  Pass 1 counts each warp's categories per plane (pass 2 redoes
// the ones and raw bits of a plane with stops, which depend on the positions'
// stream indices), one CTA barrier gives each warp its offsets, and the
// emission pass writes for every one the number of lead zeros before it in
// its stream (sc_diff_kernel turns those into the zero-run symbols) and the
// raw bits, a row's at most 32 consecutive bits or-reduced over the warp into
// at most two words.
constexpr int kScW = kScT / 32;
constexpr u64 kScWarp = 32 * kScPer;

// a word of LSB-first stream bits as stored: MSB-first within each byte, bytes in order
__device__ __forceinline__ u32 sc_word(u32 lsb_first) { return __byte_perm(__brev(lsb_first), 0, 0x0123); }

__device__ __forceinline__ void sc_flush(u32* __restrict__ raw, u64 word, u32 val, bool shared_word) {
    if (!val) return;
    if (shared_word) atomicOr(raw + word, val);
    else raw[word] = val;
}

__global__ void __launch_bounds__(kScT) sc_emit_kernel(const u64* __restrict__ m, const u8* __restrict__ neg,
                                                       const StreamDesc* __restrict__ sd, int np, int nb,
                                                       const u64* __restrict__ scoff, u64 nsc_all,
                                                       const ScOff* __restrict__ tab, u64* __restrict__ zbuf,
                                                       u32* __restrict__ raw) {
    // the sub-chunk's magnitudes (warp w: rows of 32 at sc_v[1024 w + 32 r + lane]),
    // then [plane][warp][4] counts: lead, trail, ones, raw bits
    extern __shared__ u64 sc_v[];
    u32* sc_cnt = reinterpret_cast<u32*>(sc_v + kSc);
    __shared__ int rmax_s[kScW][kScPer];  // the row's largest msb (-1: empty): rows below a plane are all lead zeros
    const u64 g = blockIdx.x;
    const int bi = sc_block(scoff, nb, g);
    const u64 j = g - scoff[bi];
    const StreamDesc d0 = sd[bi];
    const u64 lo = d0.lo + j * kSc, hi = min(d0.hi, lo + kSc);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const u64 wlo = lo + static_cast<u64>(w) * kScWarp;
    u64* v = sc_v + static_cast<u64>(w) * kScWarp + lane;  // v[32 r]: row r
    u32 negm = 0, valm = 0;
#pragma unroll 8
    for (int r = 0; r < kScPer; ++r) {
        const u64 i = wlo + static_cast<u64>(r) * 32 + lane;
        const bool ok = i < hi;
        v[32 * r] = ok ? m[i] : 0;
        if (ok) valm |= 1u << r;
        if (ok && neg && neg[i]) negm |= 1u << r;
        const int mx = __reduce_max_sync(0xffffffffu, ok ? top_bit(v[32 * r]) : -1);
        if (lane == 0) rmax_s[w][r] = mx;
    }
    __syncwarp();
    const int* rmax = rmax_s[w];
    // pass 1: category counts of this warp's positions, per plane
    for (int pi = 0; pi < np; ++pi) {
        const int p = sd[static_cast<u64>(pi) * nb + bi].plane;
        u32 nl = 0, nt = 0, no = 0;
#pragma unroll 4
        for (int r = 0; r < kScPer; ++r) {
            const bool ok = (valm >> r) & 1u;
            if (rmax[r] < p) {
                nl += __popc(__ballot_sync(0xffffffffu, ok));
                continue;
            }
            nl += __popc(__ballot_sync(0xffffffffu, ok && top_bit(v[32 * r]) <= p));
            nt += __popc(__ballot_sync(0xffffffffu, ok && top_bit(v[32 * r]) > p));
            no += __popc(__ballot_sync(0xffffffffu, ok && top_bit(v[32 * r]) == p));
        }
        if (lane == 0) {
            u32* c = sc_cnt + (pi * kScW + w) * 4;
            c[0] = nl;
            c[1] = nt;
            c[2] = no;
            c[3] = nt + no;
        }
    }
    __syncthreads();
    auto base = [&](int pi, int k) {
        u32 x = 0;
        for (int q = 0; q < w; ++q) x += sc_cnt[(pi * kScW + q) * 4 + k];
        return x;
    };
    // pass 2: planes with stops (the breakpoint plane): ones and raw bits up to the stops
    bool any_stop = false;
    for (int pi = 0; pi < np; ++pi) {
        const StreamDesc d = sd[static_cast<u64>(pi) * nb + bi];
        if (d.lstop == kFull && d.tstop == kFull) continue;
        any_stop = true;
        const int p = d.plane;
        const ScOff off = tab[static_cast<u64>(pi) * nsc_all + g];
        u64 LB = off.lead_b + base(pi, 0), TB = off.trail_b + base(pi, 1);
        u32 no = 0, nr = 0;
#pragma unroll 4
        for (int r = 0; r < kScPer; ++r) {
            const bool ok = (valm >> r) & 1u;
            if (rmax[r] < p) {
                LB += __popc(__ballot_sync(0xffffffffu, ok));
                continue;
            }
            const bool isl = ok && top_bit(v[32 * r]) <= p, ist = ok && top_bit(v[32 * r]) > p;
            const unsigned lm = __ballot_sync(0xffffffffu, isl), tm = __ballot_sync(0xffffffffu, ist);
            const u64 li = LB + __popc(lm & lt), ti = TB + __popc(tm & lt);
            const bool one = isl && top_bit(v[32 * r]) == p && li < d.lstop;
            const bool tr = ist && ti < d.tstop;
            no += __popc(__ballot_sync(0xffffffffu, one));
            nr += __popc(__ballot_sync(0xffffffffu, one || tr));
            LB += __popc(lm);
            TB += __popc(tm);
        }
        if (lane == 0) {  // fields 2, 3 only: the lead / trail counts read above stay
            sc_cnt[(pi * kScW + w) * 4 + 2] = no;
            sc_cnt[(pi * kScW + w) * 4 + 3] = nr;
        }
    }
    if (any_stop) __syncthreads();
    // emission
    for (int pi = 0; pi < np; ++pi) {
        const StreamDesc d = sd[static_cast<u64>(pi) * nb + bi];
        const int p = d.plane;
        const ScOff off = tab[static_cast<u64>(pi) * nsc_all + g];
        u64 LB = off.lead_b + base(pi, 0), TB = off.trail_b + base(pi, 1);
        u64 OB = off.ones_b + base(pi, 2);
        u64 RB = d.raw_off + off.raw_b + base(pi, 3);
        const u64 rfirst = RB >> 5;
        u64 cw = rfirst;
        u32 cv = 0;
#pragma unroll 4
        for (int r = 0; r < kScPer; ++r) {
            const bool ok = (valm >> r) & 1u;
            if (rmax[r] < p) {  // lead zeros only
                LB += __popc(__ballot_sync(0xffffffffu, ok));
                continue;
            }
            const bool isl = ok && top_bit(v[32 * r]) <= p, ist = ok && top_bit(v[32 * r]) > p;
            const unsigned lm = __ballot_sync(0xffffffffu, isl), tm = __ballot_sync(0xffffffffu, ist);
            const u64 li = LB + __popc(lm & lt), ti = TB + __popc(tm & lt);
            const bool one = isl && top_bit(v[32 * r]) == p && li < d.lstop;
            const bool tr = ist && ti < d.tstop;
            const unsigned om = __ballot_sync(0xffffffffu, one), rm = __ballot_sync(0xffffffffu, one || tr);
            if (one) {
                const u64 oi = OB + __popc(om & lt);
                zbuf[d.sym_off + oi] = li - oi;
            }
            if (rm) {
                // the row's raw bits packed LSB-first (bit k = the k-th raw position),
                // placed at the stream offset in a 64-bit window over words cw, cw + 1
                const bool bit = one ? ((negm >> r) & 1u) : (tr && ((v[32 * r] >> p) & 1u));
                const u32 pk = __reduce_or_sync(0xffffffffu, bit ? 1u << __popc(rm & lt) : 0u);
                const u64 W0 = RB >> 5;
                if (W0 != cw) {
                    if (lane == 0) sc_flush(raw, cw, sc_word(cv), cw == rfirst);
                    cw = W0;
                    cv = 0;
                }
                const u64 t = static_cast<u64>(pk) << (RB & 31);
                cv |= static_cast<u32>(t);
                if ((RB & 31) + __popc(rm) > 32) {
                    if (lane == 0) sc_flush(raw, cw, sc_word(cv), cw == rfirst);
                    cw = W0 + 1;
                    cv = static_cast<u32>(t >> 32);
                }
            }
            LB += __popc(lm);
            TB += __popc(tm);
            OB += __popc(om);
            RB += __popc(rm);
        }
        if (lane == 0) sc_flush(raw, cw, sc_word(cv), true);
    }
}

// one CTA per stream: the lead-zero counts before each one -> zero-run symbols
// (rle_extract, entropy.cpp:51-64: one run per one, then the final run)
__global__ void __launch_bounds__(256) sc_diff_kernel(const StreamDesc* __restrict__ sd,
                                                      const StreamOut* __restrict__ so, const u64* __restrict__ ncol,
                                                      const u64* __restrict__ zbuf, u64* __restrict__ syms) {
    const int st = blockIdx.x;  // blockIdx.y: 64K-symbol segments of the stream
    const u64 nsy = so[st].nsyms;
    const u64 k0 = static_cast<u64>(blockIdx.y) << 16;
    if (k0 >= nsy) return;
    const u64 no = nsy - 1, off = sd[st].sym_off, k1 = min(nsy, k0 + (u64{1} << 16));
    for (u64 k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const u64 prev = k > 0 ? zbuf[off + k - 1] : 0;
        syms[off + k] = (k < no ? zbuf[off + k] : ncol[st] - no) - prev;
    }
}

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

__host__ __device__ inline u32 log2_at_least(u32 v) {
    u32 b = 5;
    while ((1u << b) < v) ++b;
    return b;
}
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


// ---------------------------------------------------------------- per-block msb histogram
// bins 0..64 <-> msb -1..63; sizes every (plane, block) stream exactly
__global__ void msb_hist_kernel(const u64* __restrict__ m, u64 n, u64 block, u64 cpb, u64 span,
                                unsigned long long* __restrict__ hist) {
    __shared__ u32 h[65];
    for (int i = threadIdx.x; i < 65; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const u64 b = blockIdx.x / cpb, j = blockIdx.x % cpb;
    const u64 blo = b * block, bhi = min(n, blo + block);
    const u64 lo = blo + j * span, hi = min(bhi, lo + span);
    for (u64 i0 = lo; i0 < hi; i0 += blockDim.x) {
        const u64 i = i0 + threadIdx.x;
        const int bin = i < hi ? top_bit(m[i]) + 1 : -1;
        const unsigned act = __ballot_sync(0xffffffffu, bin >= 0);
        const unsigned same = __match_any_sync(0xffffffffu, bin) & act;
        if (bin >= 0 && (__ffs(same) - 1) == static_cast<int>(threadIdx.x & 31)) atomicAdd(&h[bin], __popc(same));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 65; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[b * 65 + i], static_cast<unsigned long long>(h[i]));
}

}  // namespace

std::vector<u64> msb_histogram(const u64* m, u64 n, u64 block, cudaStream_t s) {
    const u64 nb = n == 0 ? 0 : (n + block - 1) / block;
    std::vector<u64> h(nb * 65, 0);
    if (nb == 0) return h;
    const u64 span = 1 << 16;
    const u64 cpb = (block + span - 1) / span;
    DevBuf<unsigned long long> d(nb * 65, s);
    d.zero();
    msb_hist_kernel<<<static_cast<unsigned>(nb * cpb), 256, 0, s>>>(m, n, block, cpb, span, d.p);
    count_launch();
    TCB_LAUNCH();
    d2h(h.data(), d.p, nb * 65 * sizeof(u64), s);
    stream_sync(s);
    return h;
}

namespace {

// exact sizes of the full-plane stream (plane p) of one block; bounds for a breakpoint plane
struct StreamCaps {
    u64 nsyms, nraw, lead;
};
StreamCaps stream_caps(const u64* hb, int p) {
    u64 lead = 0, trail = 0;
    for (int q = -1; q <= p; ++q) lead += hb[q + 1];
    for (int q = p + 1; q < 64; ++q) trail += hb[q + 1];
    const u64 ones = hb[p + 1];
    return {lead > 0 ? ones + 1 : 0, trail + ones, lead};
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
    const u64 spb = (block + kDmSc - 1) / kDmSc;  // sub-chunks per block
    DevBuf<unsigned long long> cnt(2 * nb * spb, s);
    const unsigned grid = static_cast<unsigned>(nb * spb);
    dm_count_kernel<<<grid, kDecThreads, 0, s>>>(m, n, block, spb, last_plane, cnt.p);
    dm_scan_kernel<<<cdiv(nb, 64), 64, 0, s>>>(cnt.p, nb, spb);
    dm_decode_kernel<<<grid, kDecThreads, 0, s>>>(m, n, block, spb, last_plane, stops_dev, cnt.p, dec);
    count_launch(3);
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
    const u64 cnt[2] = {n, 0};
    DevBuf<u64> dc(2, s);
    dc.upload(cnt, 2);
    std::vector<u64> uniq(syms_host, syms_host + n);
    std::sort(uniq.begin(), uniq.end());
    const u64 distinct = static_cast<u64>(std::unique(uniq.begin(), uniq.end()) - uniq.begin());
    const u64 cap = ac_out_cap(n, ~u64{0} >> 2);
    DevBuf<u8> ent(cap, s);
    DevBuf<u64> elen(1, s);
    ac_encode(syms.p, dc.p, 2, {AcJob{0, 0, n, ~u64{0} >> 2, distinct}}, ent.p, elen.p, s);
    const u64 el = elen.to_host()[0];
    out.resize(el);
    ent.download(out.data(), el);
    stream_sync(s);
    return out;
}

// Stream layout of planes [last_plane, top_plane] x blocks: symbols, raw bits and
// entropy output sized exactly from the blocks' msb histogram (a breakpoint
// plane with stops is bounded by its full-plane sizes).
struct Layout {
    u64 nb = 0;  // blocks in the layout's range
    std::vector<StreamDesc> sd;
    std::vector<AcDesc> ad;
    std::vector<AcJob> jobs;
    u64 sym_total = 0, raw_words = 0, out_total = 0, scratch_total = 0;
};

Layout make_layout(const std::vector<u64>& hist, u64 n, u64 block, int last_plane, int top_plane,
                   const u64* stops_host, int coder, BlockRange br = {}) {
    Layout L;
    const u64 nball = n == 0 ? 0 : (n + block - 1) / block;
    const u64 b0 = std::min(br.b0, nball), b1 = std::min(br.b1, nball);
    const u64 nb = b1 > b0 ? b1 - b0 : 0;
    const int np = top_plane - last_plane + 1;
    const u64 ns = nb * static_cast<u64>(np);
    L.nb = nb;
    L.sd.resize(ns);
    L.ad.resize(ns);
    L.jobs.resize(ns);
    for (int pi = 0; pi < np; ++pi) {
        const int p = top_plane - pi;
        for (u64 b = b0; b < b1; ++b) {
            const u64 i = pi * nb + (b - b0);
            StreamDesc& d = L.sd[i];
            d.lo = b * block;
            d.hi = std::min<u64>(n, d.lo + block);
            d.plane = p;
            const bool bp = p == last_plane && stops_host != nullptr;
            d.lstop = bp ? stops_host[2 * b] : kFull;
            d.tstop = bp ? stops_host[2 * b + 1] : kFull;
            const StreamCaps c = stream_caps(hist.data() + b * 65, p);
            d.sym_off = L.sym_total;
            L.sym_total += c.nsyms;
            d.raw_off = L.raw_words * 32;
            L.raw_words += (c.nraw + 31) / 32;
            AcDesc& a = L.ad[i];
            a.sym_off = d.sym_off;
            a.out_off = L.out_total;
            a.cap = static_cast<u32>(c.nsyms + 1);
            a.fen = 0;
            a.hbits = log2_at_least(2 * a.cap);
            if (coder == 1) {
                L.out_total += rans_out_cap(c.nsyms);
                a.model_off = (L.scratch_total + 1) & ~u64{1};
                L.scratch_total = a.model_off + rans_scratch_words(c.nsyms);
            } else {
                L.out_total += ac_out_cap(c.nsyms, c.lead);
                a.model_off = 0;
            }
            L.jobs[i] = AcJob{d.sym_off, a.out_off, c.nsyms, c.lead};
        }
    }
    return L;
}

// emit + entropy coding of a layout's streams (no host round trip)
struct Coded {
    DevBuf<StreamDesc> dsd;
    DevBuf<u64> syms;
    DevBuf<u32> raw;
    DevBuf<StreamOut> so;
    DevBuf<AcDesc> dad;
    DevBuf<u8> ent;
    DevBuf<u64> elen;
    DevBuf<u32> scratch;
    DevBuf<int> err;  // the range coder's capacity flag, read with the lengths
};

// symbols and raw bits of every stream of the layout (no entropy coding)
void emit_streams(Coded& c, const Layout& L, const u64* m, const u8* neg, cudaStream_t s) {
    const u64 ns = L.sd.size();
    c.dsd = DevBuf<StreamDesc>(ns, s);
    c.dsd.upload(L.sd.data(), ns);
    c.syms = DevBuf<u64>(L.sym_total + 1, s);
    c.raw = DevBuf<u32>(L.raw_words + 1, s);
    c.raw.zero();
    c.so = DevBuf<StreamOut>(ns, s);
    {
        ProfScope pe(kEmit, s);
        // blocks of the layout (plane-major: the first nb streams are the top plane's blocks)
        const int nb = static_cast<int>(L.nb), np = static_cast<int>(ns / std::max<u64>(L.nb, 1));
        std::vector<u64> scoff(nb + 1, 0);
        for (int b = 0; b < nb; ++b) scoff[b + 1] = scoff[b] + (L.sd[b].hi - L.sd[b].lo + kSc - 1) / kSc;
        const u64 nsc = scoff[nb];
        DevBuf<u64> dsc(nb + 1, s), ncol(ns, s);
        dsc.upload(scoff.data(), nb + 1);
        DevBuf<u32> hist(nsc * 65 + 1, s);
        DevBuf<ScOff> tab(nsc * np + 1, s);
        DevBuf<u64> zbuf(L.sym_total + 1, s);
        sc_hist_kernel<<<static_cast<unsigned>(nsc), kScT, 0, s>>>(m, c.dsd.p, dsc.p, nb, hist.p);
        sc_scan_kernel<<<cdiv(ns * 32, 128), 128, 0, s>>>(m, c.dsd.p, static_cast<int>(ns), nb, dsc.p, nsc, hist.p, tab.p,
                                                  c.so.p, ncol.p);
        const size_t smem = kSc * sizeof(u64) + static_cast<size_t>(np) * kScW * 4 * sizeof(u32);
        TCB_ONCE_PER_DEVICE(cudaFuncSetAttribute(sc_emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(kSc * sizeof(u64) + 64 * kScW * 4 * sizeof(u32))));
        sc_emit_kernel<<<static_cast<unsigned>(nsc), kScT, smem, s>>>(m, neg, c.dsd.p, np, nb, dsc.p, nsc, tab.p,
                                                                      zbuf.p, c.raw.p);
        u64 maxsym = 1;
        for (const AcJob& jb : L.jobs) maxsym = std::max(maxsym, jb.sym_cap);
        sc_diff_kernel<<<dim3(static_cast<unsigned>(ns), static_cast<unsigned>(cdiv(maxsym, u64{1} << 16))), 256, 0,
                         s>>>(c.dsd.p, c.so.p, ncol.p, zbuf.p, c.syms.p);
        count_launch(4);
        TCB_LAUNCH();
    }
}

void code_streams(Coded& c, const Layout& L, const u64* m, const u8* neg, int coder, cudaStream_t s) {
    const u64 ns = L.sd.size();
    emit_streams(c, L, m, neg, s);
    c.dad = DevBuf<AcDesc>(ns, s);
    c.dad.upload(L.ad.data(), ns);
    c.ent = DevBuf<u8>(L.out_total + 1, s);
    c.elen = DevBuf<u64>(ns, s);
    if (coder == 1) {
        c.scratch = DevBuf<u32>(L.scratch_total + 2, s);
        run_rans(c.syms.p, c.so.p, c.dad.p, static_cast<int>(ns), c.ent.p, c.scratch.p, c.elen.p, s);
    } else {
        c.err = DevBuf<int>(1, s);
        c.err.zero();
        ac_encode(c.syms.p, reinterpret_cast<const u64*>(c.so.p), 2, L.jobs, c.ent.p, c.elen.p, s, c.err.p);
    }
}

struct ProbeCache {
    u64 n = 0, nb = 0;
    cudaStream_t s = nullptr;
    Layout L;
    Coded c;
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
    c->s = side;
    const u64 nb = n == 0 ? 0 : (n + block - 1) / block;
    c->nb = nb;
    if (nb == 0) return c;
    const auto hist = msb_histogram(m, n, block, side);
    c->L = make_layout(hist, n, block, 0, 63, nullptr, coder);
    code_streams(c->c, c->L, m, nullptr, coder, side);
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
        c.c.elen.download(c.el.data(), ns);
        int herr = 0;
        if (c.c.err.p) d2h(&herr, c.c.err.p, sizeof(int), c.s);
        stream_sync(c.s);
        if (herr) throw Error("entropy: device model capacity exceeded");
        for (u64 v : c.el)
            if (v == ~u64{1}) throw Error("entropy: cannot normalize rans table");
        c.ready = true;
    }
    std::vector<u64> out(c.nb);
    for (u64 b = 0; b < c.nb; ++b) out[b] = c.el[static_cast<u64>(63 - p) * c.nb + b];
    return out;
}

namespace {
// symbols + entropy coding of planes [last_plane, top_plane]; lengths on the host
struct Emitted {
    Layout L;
    Coded c;
    std::vector<u64> el;
    std::vector<StreamOut> soh;
};
bool emit_code(Emitted& E, const u64* m, const u8* neg, u64 n, u64 block, int last_plane, int top_plane,
               const u64* stops_host, int coder, cudaStream_t s, BlockRange br = {},
               const std::vector<u64>* hist_in = nullptr) {
    if (coder != 0 && coder != 1) throw Error("entropy: unknown coder");
    const u64 nball = n == 0 ? 0 : (n + block - 1) / block;
    const u64 nb = std::min(br.b1, nball) > std::min(br.b0, nball) ? std::min(br.b1, nball) - std::min(br.b0, nball) : 0;
    const int np = top_plane - last_plane + 1;
    const u64 ns = nb * static_cast<u64>(np);
    if (ns == 0 || np <= 0) return false;
    HostTrace ht_a("emit: symbols+entropy+sync");
    const auto hist = hist_in ? *hist_in : msb_histogram(m, n, block, s);
    E.L = make_layout(hist, n, block, last_plane, top_plane, stops_host, coder, br);
    code_streams(E.c, E.L, m, neg, coder, s);
    E.el.resize(ns);
    E.soh.resize(ns);
    E.c.elen.download(E.el.data(), ns);
    E.c.so.download(E.soh.data(), ns);
    int herr = 0;
    if (E.c.err.p) d2h(&herr, E.c.err.p, sizeof(int), s);
    stream_sync(s);
    if (herr) throw Error("entropy: device model capacity exceeded");
    for (u64 v : E.el)
        if (v == ~u64{1}) throw Error("entropy: cannot normalize rans table");
    if (std::getenv("TCB_AC_STATS")) {
        u64 mx = 0, tot = 0, eb = 0, rb = 0;
        for (u64 i = 0; i < ns; ++i) {
            mx = std::max(mx, E.soh[i].nsyms);
            tot += E.soh[i].nsyms;
            eb += E.el[i];
            rb += (E.soh[i].nraw + 7) / 8;
        }
        std::fprintf(stderr, "[ac stats] planes %d..%d streams %llu symbols %llu (max %llu) entropy %llu B raw %llu B\n",
                     last_plane, top_plane, (unsigned long long)ns, (unsigned long long)tot, (unsigned long long)mx,
                     (unsigned long long)eb, (unsigned long long)rb);
    }
    return true;
}
}  // namespace

EmitDev emit_planes_device(const u64* m, const u8* neg, u64 n, u64 block, int last_plane, int top_plane,
                           const u64* stops_host, int coder, cudaStream_t s, BlockRange br,
                           const std::vector<u64>* hist) {
    EmitDev out;
    Emitted E;
    if (!emit_code(E, m, neg, n, block, last_plane, top_plane, stops_host, coder, s, br, hist)) return out;
    const u64 ns = E.el.size();
    HostTrace ht_b("emit: assemble");
    std::vector<u64> off(ns);
    out.stream_bytes.resize(ns);
    u64 tot = 0;
    for (u64 i = 0; i < ns; ++i) {
        off[i] = tot;
        out.stream_bytes[i] = 4 + 4 + E.el[i] + (E.soh[i].nraw + 7) / 8;
        tot += out.stream_bytes[i];
    }
    DevBuf<u64> doff(ns, s);
    doff.upload(off.data(), ns);
    out.body = DevBuf<u8>(tot, s);
    out.size = tot;
    ProfScope pz(kEmit, s);
    assemble_kernel<<<static_cast<unsigned>(ns), 128, 0, s>>>(E.c.ent.p, E.c.dad.p, E.c.elen.p, E.c.raw.p, E.c.dsd.p,
                                                               E.c.so.p, doff.p, out.body.p);
    count_launch();
    TCB_LAUNCH();
    out.entropy_bytes = std::move(E.el);
    return out;
}

EmitResult emit_planes(const u64* m, const u8* neg, u64 n, u64 block, int last_plane, int top_plane,
                       const u64* stops_host, int coder, bool want_body, cudaStream_t s, BlockRange br) {
    EmitResult res;
    if (!want_body) {
        Emitted E;
        if (emit_code(E, m, neg, n, block, last_plane, top_plane, stops_host, coder, s, br))
            res.entropy_bytes = std::move(E.el);
        return res;
    }
    EmitDev d = emit_planes_device(m, neg, n, block, last_plane, top_plane, stops_host, coder, s, br);
    res.body.resize(d.size);
    if (d.size) d.body.download(res.body.data(), d.size);
    stream_sync(s);
    res.entropy_bytes = std::move(d.entropy_bytes);
    return res;
}


std::vector<u64> entropy_size_bounds(const u64* m, u64 n, u64 block, int plane, cudaStream_t s, BlockRange br,
                                     const std::function<void()>& launched) {
    const u64 nball = n == 0 ? 0 : (n + block - 1) / block;
    const u64 b0 = std::min(br.b0, nball), b1 = std::min(br.b1, nball);
    if (b1 <= b0) {
        if (launched) launched();
        return {};
    }
    HostTrace ht("emit: entropy size bounds");
    const auto hist = msb_histogram(m, n, block, s);
    const Layout L = make_layout(hist, n, block, plane, plane, nullptr, 0, br);
    Coded c;
    emit_streams(c, L, m, nullptr, s);
    return ac_size_bounds(c.syms.p, reinterpret_cast<const u64*>(c.so.p), 2, L.jobs, s, launched);
}

}  // namespace tcb
