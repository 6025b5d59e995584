// Exact parallel evaluation of the reference encoder's serial double sums
// (see exact.cuh for the method).  Reference loops reproduced:
//   backward_sum_sse      error_model.cpp:34-41   (kExSq, backward)
//   recalibrate_sse       error_model.cpp:54-72   (kExRecal, backward)
//   build_block stats     core_codec.cpp:131-155  (kExLead / kExTrail, per block, forward)
//   place_stops scans     core_codec.cpp:268-341  (crossing: first s >= need)
//   finalize achieved SSE core_codec.cpp:405-411  (kExDiff, backward)
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <memory>

#include "exact.cuh"
#include "terms.cuh"

namespace tcb {

namespace {

constexpr long long kBig = 1LL << 62;        // "no partial sum" sentinel for min/max
constexpr long long kLim = 1LL << 56;        // |increment| beyond any region's width: reject
constexpr long long kAMax = (1LL << 53) - 1;  // strict interior of a region, in units
constexpr long long kAMin = (1LL << 52) + 1;

struct DevSeg {
    u64 lo, hi;
    double s0, need;
    int backward;
    int pad;
};

// Summary of a run of terms for one region: per start parity pi, the total
// increment K (in units), the min / max partial increment after each nonzero
// term (kBig / -kBig when none), and the end parity (bit pi of q).
struct Fn {
    long long K0, K1, mn0, mn1, mx0, mx1;
    int q;
    int bad;
};

struct ExRec {  // pass-2 table entry for one (kind, chunk): 64 bytes
    long long K0, K1, mn0, mn1, mx0, mx1;
    int rid;
    int qbad;  // q | bad << 2
    u32 c0, c1;
};

__device__ __forceinline__ Fn fn_id() { return Fn{0, 0, kBig, kBig, -kBig, -kBig, 2, 0}; }

__device__ __forceinline__ Fn fn_then(const Fn& f, const Fn& g) {  // f first, then g
    const int m0 = f.q & 1, m1 = (f.q >> 1) & 1;
    Fn h;
    const long long gK0 = m0 ? g.K1 : g.K0, gn0 = m0 ? g.mn1 : g.mn0, gx0 = m0 ? g.mx1 : g.mx0;
    const long long gK1 = m1 ? g.K1 : g.K0, gn1 = m1 ? g.mn1 : g.mn0, gx1 = m1 ? g.mx1 : g.mx0;
    h.K0 = f.K0 + gK0;
    h.K1 = f.K1 + gK1;
    h.mn0 = min(f.mn0, f.K0 + gn0);
    h.mn1 = min(f.mn1, f.K1 + gn1);
    h.mx0 = max(f.mx0, f.K0 + gx0);
    h.mx1 = max(f.mx1, f.K1 + gx1);
    h.q = ((g.q >> m0) & 1) | (((g.q >> m1) & 1) << 1);
    h.bad = f.bad | g.bad | (llabs(h.K0) > kLim) | (llabs(h.K1) > kLim);
    if (h.bad) h.K0 = h.K1 = 0;  // keep the (discarded) arithmetic in range
    return h;
}

// Region of a running sum: e = exponent of |s| for |s| >= 2^53 (signed: the
// sign is part of the region), 52 for |s| < 2^53 (integers: exact).
__device__ __forceinline__ int region_of(double s) {
    const u64 b = static_cast<u64>(__double_as_longlong(s));
    const int e = static_cast<int>((b >> 52) & 0x7ff) - 1023;
    if (e <= 52) return 52;
    return (b >> 63) ? -e : e;
}
__device__ __forceinline__ int rexp(int rid) { return rid < 0 ? -rid : rid; }
__device__ __forceinline__ long long units_of(double s, int rid) {
    return __double2ll_rz(scalbn(s, 52 - rexp(rid)));
}
__device__ __forceinline__ double value_of(long long a, int rid) {
    return scalbn(static_cast<double>(a), rexp(rid) - 52);
}
__device__ __forceinline__ long long lo_bound(int rid) { return rid > 52 ? kAMin : -kAMax; }
__device__ __forceinline__ long long hi_bound(int rid) { return rid < 0 ? -kAMin : kAMax; }

// t / u for an integer-valued double t and u = 2^(e-52): the round-half-even
// quotient j, or at an exact tie its floor k (tie = true).  false: |t/u| is
// too large for any sum to stay in the region.
__device__ __forceinline__ bool unitize(double t, int e, long long& j, bool& tie) {
    tie = false;
    const u64 b = static_cast<u64>(__double_as_longlong(t));
    const bool neg = b >> 63;
    const int E = static_cast<int>((b >> 52) & 0x7ff) - 1075;
    const u64 M = (b & ((u64{1} << 52) - 1)) | (u64{1} << 52);
    const int sh = (e - 52) - E;
    if (sh <= 0) {
        if (sh < -8) return false;
        const long long q = static_cast<long long>(M << (-sh));
        j = neg ? -q : q;
        return true;
    }
    if (sh >= 54) {  // |t| < u/2
        j = 0;
        return true;
    }
    const u64 qq = M >> sh, rem = M & ((u64{1} << sh) - 1), half = u64{1} << (sh - 1);
    if (rem == half) {
        tie = true;
        j = neg ? -static_cast<long long>(qq) - 1 : static_cast<long long>(qq);
        return true;
    }
    const long long r = static_cast<long long>(qq) + (rem > half ? 1 : 0);
    j = neg ? -r : r;
    return true;
}

__device__ __forceinline__ void fn_push(Fn& f, long long j, bool tie) {
    const int p0 = f.q & 1, p1 = (f.q >> 1) & 1;
    const int jb = static_cast<int>(j & 1);
    long long i0 = j, i1 = j;
    int n0, n1;
    if (tie) {  // a + k + 1/2 -> the even neighbour
        i0 += (p0 ^ jb);
        i1 += (p1 ^ jb);
        n0 = n1 = 0;
    } else {
        n0 = p0 ^ jb;
        n1 = p1 ^ jb;
    }
    f.K0 += i0;
    f.K1 += i1;
    f.mn0 = min(f.mn0, f.K0);
    f.mn1 = min(f.mn1, f.K1);
    f.mx0 = max(f.mx0, f.K0);
    f.mx1 = max(f.mx1, f.K1);
    f.q = n0 | (n1 << 1);
    if (llabs(f.K0) > kLim || llabs(f.K1) > kLim) {
        f.bad = 1;
        f.K0 = f.K1 = 0;
    }
}

__device__ __forceinline__ void fn_term(Fn& f, double t, int e) {
    if (t == 0.0 || f.bad) return;  // s + 0 = s exactly
    long long j;
    bool tie;
    if (!unitize(t, e, j, tie)) {
        f.bad = 1;
        f.K0 = f.K1 = 0;
        return;
    }
    fn_push(f, j, tie);
}

// term of element value v (and decoded value d) for a kind; cat0/cat1: the
// element's category counts (see ExOut)
__device__ __forceinline__ double ex_term(int term, int p, u64 v, u64 d, u32& cat0, u32& cat1) {
    switch (term) {
        case kExLead: {
            const int tb = top_bit64(v);
            cat0 = tb <= p;
            cat1 = tb == p;
            return tb == p ? t_lead_gain(v, p) : 0.0;
        }
        case kExTrail: {
            const int tb = top_bit64(v);
            cat0 = 0;
            cat1 = tb > p;
            return tb > p ? t_trail_gain(v, p) : 0.0;
        }
        case kExBoth: {
            const int tb = top_bit64(v);
            cat0 = tb <= p;
            cat1 = tb > p;
            return tb > p ? t_trail_gain(v, p) : (tb == p ? t_lead_gain(v, p) : 0.0);
        }
        case kExSq: cat0 = cat1 = 0; return t_insig2(v);
        case kExRecal: cat0 = cat1 = 0; return t_recal(v, p);
        default: cat0 = cat1 = 0; return t_diff2(v, d);
    }
}

__device__ __forceinline__ u64 elem_index(const DevSeg& g, u64 q) { return g.backward ? g.hi - 1 - q : g.lo + q; }

__device__ __forceinline__ int seg_of(const u64* choff, int nseg, u64 c) {
    int lo = 0, hi = nseg - 1;  // last g with choff[g] <= c
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(choff + mid) <= c) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ Fn shfl_fn(const Fn& f, int src, bool up_by) {
    (void)up_by;
    Fn g;
    g.K0 = __shfl_sync(0xffffffffu, f.K0, src);
    g.K1 = __shfl_sync(0xffffffffu, f.K1, src);
    g.mn0 = __shfl_sync(0xffffffffu, f.mn0, src);
    g.mn1 = __shfl_sync(0xffffffffu, f.mn1, src);
    g.mx0 = __shfl_sync(0xffffffffu, f.mx0, src);
    g.mx1 = __shfl_sync(0xffffffffu, f.mx1, src);
    g.q = __shfl_sync(0xffffffffu, f.q, src);
    g.bad = __shfl_sync(0xffffffffu, f.bad, src);
    return g;
}

// inclusive warp scan of the composition (lane order = sequence order)
__device__ __forceinline__ Fn warp_scan_fn(Fn f) {
    const int lane = threadIdx.x & 31;
    for (int o = 1; o < 32; o <<= 1) {
        const Fn g = shfl_fn(f, lane >= o ? lane - o : lane, true);
        if (lane >= o) f = fn_then(g, f);
    }
    return f;
}

// ---------------------------------------------------------------- passes 1 and 2
// Work item = (chunk, kind), one warp each; the warps of a CTA take
// consecutive items, i.e. the kinds of one chunk, so a chunk's magnitudes are
// read from DRAM once and from L1/L2 by the other kinds.  Lane l owns the
// contiguous positions [l * LPE, (l + 1) * LPE) of the chunk, so its run of
// terms is a contiguous piece of the serial order and the warp combines the
// lanes' functions in lane order.
constexpr int kExWarps = 8;

// element positions of one lane: term value or 0, category counts; TERM is
// resolved once per item (no per-element switch)
template <int TERM, class F>
__device__ __forceinline__ void lane_terms(const u64* __restrict__ m, const u64* __restrict__ dec, const DevSeg& sg,
                                           u64 q0, int cnt, int p, F&& f) {
    for (int i = 0; i < cnt; ++i) {
        const u64 idx = elem_index(sg, q0 + i);
        const u64 v = __ldg(m + idx);
        if constexpr (TERM == kExLead) {
            const int tb = top_bit64(v);
            f(tb == p ? t_lead_gain(v, p) : 0.0, tb <= p, tb == p, tb == p);
        } else if constexpr (TERM == kExTrail) {
            const int tb = top_bit64(v);
            f(tb > p ? t_trail_gain(v, p) : 0.0, 0u, tb > p, tb > p);
        } else if constexpr (TERM == kExBoth) {
            const int tb = top_bit64(v);
            const bool tr = tb > p;
            f(tr ? t_trail_gain(v, p) : (tb == p ? t_lead_gain(v, p) : 0.0), !tr, tr, tb >= p);
        } else if constexpr (TERM == kExSq) {
            f(t_insig2(v), 0u, 0u, v != 0);
        } else if constexpr (TERM == kExRecal) {
            f(t_recal(v, p), 0u, 0u, true);
        } else {
            f(t_diff2(v, __ldg(dec + idx)), 0u, 0u, true);
        }
    }
}

struct ItemGeom {
    int g;
    u64 q0;  // first position of this lane
    int cnt; // positions of this lane
};
template <int LPE>
__device__ __forceinline__ ItemGeom item_geom(const DevSeg* __restrict__ segs, int nseg, const u64* __restrict__ choff,
                                              u64 c, DevSeg& sg) {
    constexpr u64 C = 32ull * LPE;
    ItemGeom ig;
    ig.g = seg_of(choff, nseg, c);
    sg = segs[ig.g];
    const u64 len = sg.hi - sg.lo;
    ig.q0 = (c - choff[ig.g]) * C + static_cast<u64>(threadIdx.x & 31) * LPE;
    ig.cnt = ig.q0 >= len ? 0 : static_cast<int>(min(static_cast<u64>(LPE), len - ig.q0));
    return ig;
}

template <int LPE>
__global__ void __launch_bounds__(32 * kExWarps) ex_approx_kernel(const u64* __restrict__ m, const u64* __restrict__ dec,
                                                                  const DevSeg* __restrict__ segs, int nseg,
                                                                  const u64* __restrict__ choff,
                                                                  const ExKind* __restrict__ kinds, int nk, u64 nch,
                                                                  double* __restrict__ A) {
    const u64 item = static_cast<u64>(blockIdx.x) * kExWarps + (threadIdx.x >> 5);
    if (item >= nch * nk) return;
    const u64 c = item / nk;
    const int k = static_cast<int>(item % nk);
    DevSeg sg;
    const ItemGeom ig = item_geom<LPE>(segs, nseg, choff, c, sg);
    const ExKind kd = kinds[k];
    double acc = 0.0;
    auto add = [&](double t, u32, u32, bool) { acc += t; };
    switch (kd.term) {
        case kExLead: lane_terms<kExLead>(m, dec, sg, ig.q0, ig.cnt, kd.plane, add); break;
        case kExTrail: lane_terms<kExTrail>(m, dec, sg, ig.q0, ig.cnt, kd.plane, add); break;
        case kExBoth: lane_terms<kExBoth>(m, dec, sg, ig.q0, ig.cnt, kd.plane, add); break;
        case kExSq: lane_terms<kExSq>(m, dec, sg, ig.q0, ig.cnt, kd.plane, add); break;
        case kExRecal: lane_terms<kExRecal>(m, dec, sg, ig.q0, ig.cnt, kd.plane, add); break;
        default: lane_terms<kExDiff>(m, dec, sg, ig.q0, ig.cnt, kd.plane, add); break;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) A[static_cast<u64>(k) * nch + c] = acc;
}

// exclusive prefix (plus s0) of the approximate chunk sums of each (kind, segment)
__global__ void __launch_bounds__(1024) ex_scan_kernel(const DevSeg* __restrict__ segs, int nseg,
                                                       const u64* __restrict__ choff, u64 nch,
                                                       const double* __restrict__ A, double* __restrict__ P) {
    __shared__ double sh[32];
    __shared__ double carry_s;
    const int k = blockIdx.x / nseg, g = blockIdx.x % nseg;
    const u64 b0 = choff[g], b1 = choff[g + 1];
    const double* a = A + static_cast<u64>(k) * nch;
    double* p = P + static_cast<u64>(k) * nch;
    if (threadIdx.x == 0) carry_s = segs[g].s0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (u64 t0 = b0; t0 < b1; t0 += blockDim.x) {
        const u64 i = t0 + threadIdx.x;
        const double x = i < b1 ? a[i] : 0.0;
        double y = x;
        for (int o = 1; o < 32; o <<= 1) {
            const double z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        if (lane == 31) sh[w] = y;
        __syncthreads();
        if (w == 0) {
            double z = lane < static_cast<int>(blockDim.x >> 5) ? sh[lane] : 0.0;
            for (int o = 1; o < 32; o <<= 1) {
                const double zz = __shfl_up_sync(0xffffffffu, z, o);
                if (lane >= o) z += zz;
            }
            sh[lane] = z;  // inclusive warp totals
        }
        __syncthreads();
        const double carry = carry_s;
        const double excl = carry + (w > 0 ? sh[w - 1] : 0.0) + (y - x);
        if (i < b1) p[i] = excl;
        __syncthreads();
        if (threadIdx.x == 0) carry_s = carry + sh[(blockDim.x >> 5) - 1];
        __syncthreads();
    }
}

template <int LPE>
__global__ void __launch_bounds__(32 * kExWarps) ex_fn_kernel(const u64* __restrict__ m, const u64* __restrict__ dec,
                                                              const DevSeg* __restrict__ segs, int nseg,
                                                              const u64* __restrict__ choff,
                                                              const ExKind* __restrict__ kinds, int nk, u64 nch,
                                                              const double* __restrict__ P, ExRec* __restrict__ out) {
    const u64 item = static_cast<u64>(blockIdx.x) * kExWarps + (threadIdx.x >> 5);
    if (item >= nch * nk) return;
    const int lane = threadIdx.x & 31;
    const u64 c = item / nk;
    const int k = static_cast<int>(item % nk);
    DevSeg sg;
    const ItemGeom ig = item_geom<LPE>(segs, nseg, choff, c, sg);
    const ExKind kd = kinds[k];
    const int rid = region_of(P[static_cast<u64>(k) * nch + c]);
    const int e = rexp(rid);
    Fn f = fn_id();
    u32 x0 = 0, x1 = 0;
    auto push = [&](double t, u32 a0, u32 a1, bool nz) {
        x0 += a0;
        x1 += a1;
        if (nz) fn_term(f, t, e);
    };
    switch (kd.term) {
        case kExLead: lane_terms<kExLead>(m, dec, sg, ig.q0, ig.cnt, kd.plane, push); break;
        case kExTrail: lane_terms<kExTrail>(m, dec, sg, ig.q0, ig.cnt, kd.plane, push); break;
        case kExBoth: lane_terms<kExBoth>(m, dec, sg, ig.q0, ig.cnt, kd.plane, push); break;
        case kExSq: lane_terms<kExSq>(m, dec, sg, ig.q0, ig.cnt, kd.plane, push); break;
        case kExRecal: lane_terms<kExRecal>(m, dec, sg, ig.q0, ig.cnt, kd.plane, push); break;
        default: lane_terms<kExDiff>(m, dec, sg, ig.q0, ig.cnt, kd.plane, push); break;
    }
    // ordered reduction: lane l (aligned to 2o) absorbs lanes [l + o, l + 2o)
    for (int o = 1; o < 32; o <<= 1) {
        const Fn h = shfl_fn(f, (lane + o) & 31, false);
        if ((lane & (2 * o - 1)) == 0) f = fn_then(f, h);
    }
    for (int o = 16; o > 0; o >>= 1) {
        x0 += __shfl_xor_sync(0xffffffffu, x0, o);
        x1 += __shfl_xor_sync(0xffffffffu, x1, o);
    }
    if (lane == 0) {
        ExRec r;
        r.K0 = f.K0;
        r.K1 = f.K1;
        r.mn0 = f.mn0;
        r.mn1 = f.mn1;
        r.mx0 = f.mx0;
        r.mx1 = f.mx1;
        r.rid = rid;
        r.qbad = f.q | (f.bad << 2);
        r.c0 = x0;
        r.c1 = x1;
        out[static_cast<u64>(k) * nch + c] = r;
    }
}

// ---------------------------------------------------------------- the walk
struct WalkState {
    double s;
    u64 c0, c1;
    int crossed;
};

// Warp-cooperative exact resolution of processing positions [q, q1) of one
// segment: 8-term functions per lane for the current region, composed by a
// warp scan; the lanes before the first rejected one are applied at once, the
// rejected lane's terms are added serially.
__device__ void ex_fine(const u64* __restrict__ m, const u64* __restrict__ dec, const ExKind kd, const DevSeg& sg,
                        u64 q, u64 q1, WalkState& st) {
    const int lane = threadIdx.x & 31;
    const bool xing = sg.need < HUGE_VAL;
    while (q < q1 && !st.crossed) {
        const int rid = region_of(st.s);
        const long long a = units_of(st.s, rid);
        const int pi0 = static_cast<int>(a & 1);
        const u64 lb = q + 8ull * lane, le = min(lb + 8, q1);
        Fn f = fn_id();
        u32 x0 = 0, x1 = 0;
        for (u64 qq = lb; qq < le; ++qq) {
            const u64 idx = elem_index(sg, qq);
            u32 a0, a1;
            const double t = ex_term(kd.term, kd.plane, m[idx], dec ? dec[idx] : 0, a0, a1);
            x0 += a0;
            x1 += a1;
            fn_term(f, t, rexp(rid));
        }
        const Fn incl = warp_scan_fn(f);
        Fn ex = shfl_fn(incl, lane > 0 ? lane - 1 : 0, true);
        if (lane == 0) ex = fn_id();
        const long long al = a + (pi0 ? ex.K1 : ex.K0);
        const int pil = (ex.q >> pi0) & 1;
        const long long rn = pil ? f.mn1 : f.mn0, rx = pil ? f.mx1 : f.mx0;
        bool ok = !f.bad && !ex.bad && al + rn >= lo_bound(rid) && al + rx <= hi_bound(rid);
        if (ok && xing && rx > -kBig && value_of(al + rx, rid) >= sg.need) ok = false;
        const unsigned bm = __ballot_sync(0xffffffffu, !ok);
        const int b = bm ? __ffs(bm) - 1 : 32;
        if (b > 0) {
            const long long inc = __shfl_sync(0xffffffffu, pi0 ? incl.K1 : incl.K0, b - 1);
            st.s = value_of(a + inc, rid);
            u32 y0 = lane < b ? x0 : 0, y1 = lane < b ? x1 : 0;
            for (int o = 16; o > 0; o >>= 1) {
                y0 += __shfl_xor_sync(0xffffffffu, y0, o);
                y1 += __shfl_xor_sync(0xffffffffu, y1, o);
            }
            st.c0 += y0;
            st.c1 += y1;
        }
        if (b == 32) {
            q += 256;
            continue;
        }
        // lane b's terms one at a time (every lane redundantly: identical state)
        const u64 sb = q + 8ull * b, se = min(sb + 8, q1);
        for (u64 qq = sb; qq < se; ++qq) {
            const u64 idx = elem_index(sg, qq);
            u32 a0, a1;
            const double t = ex_term(kd.term, kd.plane, m[idx], dec ? dec[idx] : 0, a0, a1);
            st.c0 += a0;
            st.c1 += a1;
            st.s = __dadd_rn(st.s, t);
            if (xing && st.s >= sg.need) {
                st.crossed = 1;
                break;
            }
        }
        q = se;
    }
}

template <int LPE>
__global__ void __launch_bounds__(128) ex_walk_kernel(const u64* __restrict__ m, const u64* __restrict__ dec,
                                                      const DevSeg* __restrict__ segs, int nseg,
                                                      const u64* __restrict__ choff, const ExKind* __restrict__ kinds,
                                                      int njobs, u64 nch, const ExRec* __restrict__ recs,
                                                      ExOut* __restrict__ out) {
    constexpr u64 C = 32ull * LPE;
    const int job = static_cast<int>((static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    if (job >= njobs) return;
    const int lane = threadIdx.x & 31;
    const int k = job / nseg, g = job % nseg;
    const ExKind kd = kinds[k];
    const DevSeg sg = segs[g];
    const bool xing = sg.need < HUGE_VAL;
    WalkState st{sg.s0, 0, 0, 0};
    const u64 len = sg.hi - sg.lo;
    if (xing && st.s >= sg.need) {
        st.crossed = 1;
    } else if (recs && len > 0) {
        const u64 nc = (len + C - 1) / C;
        const ExRec* rk = recs + static_cast<u64>(k) * nch + choff[g];
        for (u64 c = 0; c < nc && !st.crossed;) {
            const int rid = region_of(st.s);
            const long long a = units_of(st.s, rid);
            const int pi0 = static_cast<int>(a & 1);
            const u64 cc = c + lane;
            const bool have = cc < nc;
            ExRec r;
            if (have) r = rk[cc];
            Fn f = fn_id();
            bool pre = false;
            if (have) {
                f = Fn{r.K0, r.K1, r.mn0, r.mn1, r.mx0, r.mx1, r.qbad & 3, (r.qbad >> 2) & 1};
                pre = r.rid == rid && !f.bad;
                if (!pre) f = fn_id();
            } else {
                r.c0 = r.c1 = 0;
            }
            const Fn incl = warp_scan_fn(f);
            Fn ex = shfl_fn(incl, lane > 0 ? lane - 1 : 0, true);
            if (lane == 0) ex = fn_id();
            const long long al = a + (pi0 ? ex.K1 : ex.K0);
            const int pil = (ex.q >> pi0) & 1;
            const long long rn = pil ? f.mn1 : f.mn0, rx = pil ? f.mx1 : f.mx0;
            bool ok = pre && !ex.bad && al + rn >= lo_bound(rid) && al + rx <= hi_bound(rid);
            if (ok && xing && rx > -kBig && value_of(al + rx, rid) >= sg.need) ok = false;
            const unsigned bm = __ballot_sync(0xffffffffu, !ok);
            const int b = bm ? __ffs(bm) - 1 : 32;
            if (b > 0) {
                const long long inc = __shfl_sync(0xffffffffu, pi0 ? incl.K1 : incl.K0, b - 1);
                st.s = value_of(a + inc, rid);
                u32 y0 = lane < b ? r.c0 : 0, y1 = lane < b ? r.c1 : 0;
                for (int o = 16; o > 0; o >>= 1) {
                    y0 += __shfl_xor_sync(0xffffffffu, y0, o);
                    y1 += __shfl_xor_sync(0xffffffffu, y1, o);
                }
                st.c0 += y0;
                st.c1 += y1;
            }
            c += b;
            if (b < 32 && c < nc) {
                ex_fine(m, dec, kd, sg, c * C, min((c + 1) * C, len), st);
                c += 1;
            }
        }
    } else if (len > 0) {
        ex_fine(m, dec, kd, sg, 0, len, st);
    }
    if (lane == 0) out[job] = ExOut{st.s, st.c0, st.c1, st.crossed};
}

// one thread per job: the plain serial loop (verification only)
__global__ void ex_serial_kernel(const u64* __restrict__ m, const u64* __restrict__ dec,
                                 const DevSeg* __restrict__ segs, int nseg, const ExKind* __restrict__ kinds,
                                 int njobs, ExOut* __restrict__ out) {
    const int job = static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x);
    if (job >= njobs) return;
    const int k = job / nseg, g = job % nseg;
    const ExKind kd = kinds[k];
    const DevSeg sg = segs[g];
    const bool xing = sg.need < HUGE_VAL;
    ExOut o{sg.s0, 0, 0, 0};
    if (xing && o.sum >= sg.need) {
        o.crossed = 1;
    } else {
        for (u64 q = 0; q < sg.hi - sg.lo; ++q) {
            const u64 idx = elem_index(sg, q);
            u32 a0, a1;
            const double t = ex_term(kd.term, kd.plane, m[idx], dec ? dec[idx] : 0, a0, a1);
            o.c0 += a0;
            o.c1 += a1;
            o.sum = __dadd_rn(o.sum, t);
            if (xing && o.sum >= sg.need) {
                o.crossed = 1;
                break;
            }
        }
    }
    out[job] = o;
}

// ---------------------------------------------------------------- plane statistics, lane = plane
// build_block's statistics for up to 32 consecutive planes at once: one warp
// streams a chunk's magnitudes once (every load a broadcast) and lane l owns
// plane p_top - l, evaluating only its own lead / trail terms.  Kinds are
// (lead, trail) of each plane in lane order: k = 2 l + {0, 1}.
//
// Compact transducer state: until the first exact tie both start parities
// follow the same path (A, with its min / max); the tie sends them to
// neighbouring values (k1 or k1 + 1 depending on the start parity) and leaves
// an even result, after which the path is again parity independent (B).
struct CFn {
    long long A, mnA, mxA, k1, B, mnB, mxB;
    int tie, bpar, bad;
};
__device__ __forceinline__ CFn cfn_id() { return CFn{0, kBig, -kBig, 0, 0, 0, 0, 0, 0, 0}; }
// unitize() in floating point: y = t / u exactly (u = 2^(e-52) = 1 / scale), the
// round-half-even increment by one conversion, a tie when y - j is exactly 1/2
// (then j = floor(y), as unitize returns); |y| >= 2^61 is unitize's rejection.
__device__ __forceinline__ bool unit_fp(double t, double scale, long long& j, bool& tie) {
    const double y = t * scale;
    if (fabs(y) >= 0x1p61) return false;
    j = __double2ll_rn(y);
    const double d = y - static_cast<double>(j);  // exact: |d| <= 1/2
    tie = fabs(d) == 0.5;
    if (tie && d < 0.0) j -= 1;
    return true;
}
__device__ __forceinline__ void cfn_push(CFn& f, long long j, bool tie) {
    if (!f.tie) {
        if (!tie) {
            f.A += j;
            f.mnA = min(f.mnA, f.A);
            f.mxA = max(f.mxA, f.A);
        } else {
            f.tie = 1;
            f.k1 = j;
        }
    } else {
        const int jb = static_cast<int>(j & 1);
        f.B += tie ? j + ((f.bpar ^ jb) & 1) : j;
        f.bpar = tie ? 0 : (f.bpar ^ jb);
        f.mnB = min(f.mnB, f.B);
        f.mxB = max(f.mxB, f.B);
    }
    if (llabs(f.A) > kLim || llabs(f.B) > kLim) f.bad = 1;
}
__device__ __forceinline__ ExRec cfn_rec(const CFn& f, int rid, u32 c0, u32 c1) {
    ExRec r;
    r.rid = rid;
    r.c0 = c0;
    r.c1 = c1;
    if (f.bad) {
        r.K0 = r.K1 = 0;
        r.mn0 = r.mn1 = kBig;
        r.mx0 = r.mx1 = -kBig;
        r.qbad = 2 | 4;
        return r;
    }
    if (!f.tie) {
        r.K0 = r.K1 = f.A;
        r.mn0 = r.mn1 = f.mnA;
        r.mx0 = r.mx1 = f.mxA;
        const int ap = static_cast<int>(f.A & 1);
        r.qbad = ap | ((1 ^ ap) << 1);
        return r;
    }
    const int ak = static_cast<int>((f.A ^ f.k1) & 1);
    const long long t0 = f.A + f.k1 + (ak & 1), t1 = f.A + f.k1 + ((1 ^ ak) & 1);  // value after the tie
    r.K0 = t0 + f.B;
    r.K1 = t1 + f.B;
    r.mn0 = min(f.mnA, t0 + f.mnB);
    r.mn1 = min(f.mnA, t1 + f.mnB);
    r.mx0 = max(f.mxA, t0 + f.mxB);
    r.mx1 = max(f.mxA, t1 + f.mxB);
    r.qbad = f.bpar | (f.bpar << 1);
    return r;
}

// CFn -> the composable Fn (the same fields cfn_rec writes)
__device__ __forceinline__ Fn cfn_fn(const CFn& f) {
    const ExRec r = cfn_rec(f, 0, 0, 0);
    return Fn{r.K0, r.K1, r.mn0, r.mn1, r.mx0, r.mx1, r.qbad & 3, (r.qbad >> 2) & 1};
}
__device__ __forceinline__ Fn fn_shfl_down(const Fn& f, int o) {
    Fn g;
    g.K0 = __shfl_down_sync(0xffffffffu, f.K0, o);
    g.K1 = __shfl_down_sync(0xffffffffu, f.K1, o);
    g.mn0 = __shfl_down_sync(0xffffffffu, f.mn0, o);
    g.mn1 = __shfl_down_sync(0xffffffffu, f.mn1, o);
    g.mx0 = __shfl_down_sync(0xffffffffu, f.mx0, o);
    g.mx1 = __shfl_down_sync(0xffffffffu, f.mx1, o);
    g.q = __shfl_down_sync(0xffffffffu, f.q, o);
    g.bad = __shfl_down_sync(0xffffffffu, f.bad, o);
    return g;
}
// the lanes' functions composed in lane order (lane 0 first); valid in lane 0
__device__ __forceinline__ Fn fn_warp_compose(Fn f) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const Fn g = fn_shfl_down(f, o);
        if ((lane & (2 * o - 1)) == 0) f = fn_then(f, g);
    }
    return f;
}
__device__ __forceinline__ ExRec fn_rec(const Fn& f, int rid, u32 c0, u32 c1) {
    ExRec r;
    r.K0 = f.K0;
    r.K1 = f.K1;
    r.mn0 = f.mn0;
    r.mn1 = f.mn1;
    r.mx0 = f.mx0;
    r.mx1 = f.mx1;
    r.rid = rid;
    r.qbad = (f.q & 3) | (f.bad << 2);
    r.c0 = c0;
    r.c1 = c1;
    return r;
}

// One warp per 2048-element chunk, staged in shared memory; lane l takes the
// contiguous run [64 l, 64 l + 64) and the planes one after another: its run's
// lead and trail functions (PASS 1) or approximate sums (PASS 0) per plane,
// then the 32 runs are composed (summed) in lane order.  Per plane a lane
// touches only its elements with msb >= p, so the work follows the active
// (element, plane) pairs instead of one element at a time across 32 plane lanes.
constexpr int kPlRun = 64, kPlPad = kPlRun + 1;
template <int PASS>
__global__ void __launch_bounds__(128) ex_plane_kernel(const u64* __restrict__ m, const DevSeg* __restrict__ segs,
                                                       int nseg, const u64* __restrict__ choff, int p_top, int np,
                                                       u64 nch, double* __restrict__ A, const double* __restrict__ P,
                                                       ExRec* __restrict__ out) {
    constexpr u64 C = 2048;
    extern __shared__ u64 ex_sv[];  // 4 warps x 32 runs x kPlPad
    const u64 c = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (c >= nch) return;
    const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & 3;
    const int g = seg_of(choff, nseg, c);
    const DevSeg sg = segs[g];
    const u64 lo = sg.lo + (c - choff[g]) * C;
    const int cnt = static_cast<int>(min(C, sg.hi - lo));
    u64* v = ex_sv + w * (32 * kPlPad);
    for (int e = lane; e < static_cast<int>(C); e += 32) v[(e >> 6) * kPlPad + (e & 63)] = e < cnt ? __ldg(m + lo + e) : 0;
    __syncwarp();
    const u64* mine = v + lane * kPlPad;
    const int n_mine = max(0, min(kPlRun, cnt - lane * kPlRun));
    int tmax = -1;  // the run's largest msb: planes above it see only lead zeros
    for (int i = 0; i < n_mine; ++i) tmax = max(tmax, top_bit64(mine[i]));
    for (int l = 0; l < np; ++l) {
        const int p = p_top - l;
        // the lead / trail gains share one form (terms.cuh):
        //   t = (double(a) - c)^2 - sig2(m, p),  trail (msb > p): a = m mod 2^(p+1), c = 2^p
        //                                        lead (msb == p): a = m,            c = 0
        const int pc = p < 0 ? 0 : p;
        const u64 mask_p = pc == 0 ? 0 : (u64{1} << pc) - 1;
        const u64 mask_p1 = pc >= 63 ? ~u64{0} : (u64{1} << (pc + 1)) - 1;
        const double half_p = pc == 0 ? 0.0 : __ull2double_rn(u64{1} << (pc - 1));
        const double c_p = __ull2double_rn(u64{1} << (pc > 63 ? 63 : pc));
        double aL = 0.0, aT = 0.0;
        CFn fL = cfn_id(), fT = cfn_id();
        int rL = 52, rT = 52;
        double sL = 1.0, sT = 1.0;  // 2^(52 - e) of each function's region
        if (PASS == 1) {
            rL = region_of(P[static_cast<u64>(2 * l) * nch + c]);
            rT = region_of(P[static_cast<u64>(2 * l + 1) * nch + c]);
            sL = scalbn(1.0, 52 - rexp(rL));
            sT = scalbn(1.0, 52 - rexp(rT));
        }
        u32 nle = 0, none = 0, ntr = 0;
        if (tmax >= p) {
            for (int i = 0; i < n_mine; ++i) {
                const u64 x = mine[i];
                const int tb = top_bit64(x);
                if (tb < p) continue;
                const bool tr = tb > p;
                none += !tr;
                ntr += tr;
                const double x0 = __dsub_rn(__ull2double_rn(tr ? (x & mask_p1) : x), tr ? c_p : 0.0);
                const double r0 = __dsub_rn(__ull2double_rn(x & mask_p), half_p);
                const double t = __dsub_rn(__dmul_rn(x0, x0), pc == 0 ? 0.0 : __dmul_rn(r0, r0));
                if (PASS == 0) {
                    aT += tr ? t : 0.0;
                    aL += tr ? 0.0 : t;
                } else if (t != 0.0) {
                    long long j = 0;
                    bool tie = false;
                    const bool ok = unit_fp(t, tr ? sT : sL, j, tie);
                    if (tr) {
                        if (!ok) fT.bad = 1;
                        else if (!fT.bad) cfn_push(fT, j, tie);
                    } else {
                        if (!ok) fL.bad = 1;
                        else if (!fL.bad) cfn_push(fL, j, tie);
                    }
                }
            }
        }
        nle = static_cast<u32>(n_mine) - ntr;  // lead positions: msb <= p
        if (PASS == 0) {
            for (int o = 16; o > 0; o >>= 1) {
                aL += __shfl_down_sync(0xffffffffu, aL, o);
                aT += __shfl_down_sync(0xffffffffu, aT, o);
            }
            if (lane == 0) {
                A[static_cast<u64>(2 * l) * nch + c] = aL;
                A[static_cast<u64>(2 * l + 1) * nch + c] = aT;
            }
        } else {
            const Fn FL = fn_warp_compose(cfn_fn(fL));
            const Fn FT = fn_warp_compose(cfn_fn(fT));
            for (int o = 16; o > 0; o >>= 1) {
                nle += __shfl_down_sync(0xffffffffu, nle, o);
                none += __shfl_down_sync(0xffffffffu, none, o);
                ntr += __shfl_down_sync(0xffffffffu, ntr, o);
            }
            if (lane == 0) {
                out[static_cast<u64>(2 * l) * nch + c] = fn_rec(FL, rL, nle, none);
                out[static_cast<u64>(2 * l + 1) * nch + c] = fn_rec(FT, rT, 0, ntr);
            }
        }
    }
}

// Sampled estimate of the residual after each plane (PlaneStatsJob::approx_residuals):
// runs of 256 consecutive elements, one in every kResStride, over [lo, hi).
constexpr u64 kResRun = 256, kResStride = 64;
__global__ void __launch_bounds__(256) ex_resid_kernel(const u64* __restrict__ m, u64 lo, u64 hi, int p_top, int np,
                                                       double* __restrict__ res) {
    double acc[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) acc[l] = 0.0;
    const u64 nrun = (hi - lo + kResRun - 1) / kResRun;
    for (u64 r = static_cast<u64>(blockIdx.x) * kResStride; r < nrun; r += static_cast<u64>(gridDim.x) * kResStride) {
        const u64 i = lo + r * kResRun + threadIdx.x;
        if (i >= hi) continue;
        const u64 v = m[i];
        const int tb = top_bit64(v);
        const double vd = __ull2double_rn(v);
        const double sq = vd * vd;
#pragma unroll
        for (int l = 0; l < 32; ++l) {
            const int p = p_top - l;
            if (l >= np) break;
            double t;
            if (tb < p) {
                t = sq;
            } else if (p == 0) {
                t = 0.0;
            } else {
                const double x = __ull2double_rn(v & ((u64{1} << p) - 1)) - __ull2double_rn(u64{1} << (p - 1));
                t = x * x;
            }
            acc[l] += t;
        }
    }
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int l = 0; l < 32; ++l) {
        if (l >= np) break;
        double x = acc[l];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) atomicAdd(res + l, x);
    }
}

struct Prepared {
    std::vector<DevSeg> hs;
    std::vector<u64> choff;
    DevBuf<DevSeg> segs;
    DevBuf<u64> dch;
    DevBuf<ExKind> dk;
    u64 nch = 0, maxlen = 0;
};

Prepared prepare(const std::vector<ExSeg>& segs, const std::vector<ExKind>& kinds, u64 C, cudaStream_t s) {
    Prepared p;
    p.hs.resize(segs.size());
    p.choff.assign(segs.size() + 1, 0);
    for (std::size_t g = 0; g < segs.size(); ++g) {
        const ExSeg& e = segs[g];
        if (e.hi < e.lo) throw Error("exact sum: bad segment");
        p.hs[g] = DevSeg{e.lo, e.hi, e.s0, e.need, e.backward, 0};
        const u64 len = e.hi - e.lo;
        p.maxlen = std::max(p.maxlen, len);
        p.choff[g + 1] = p.choff[g] + (len + C - 1) / C;
    }
    p.nch = p.choff.back();
    p.segs = DevBuf<DevSeg>(segs.size(), s);
    p.segs.upload(p.hs.data(), segs.size());
    p.dch = DevBuf<u64>(segs.size() + 1, s);
    p.dch.upload(p.choff.data(), segs.size() + 1);
    p.dk = DevBuf<ExKind>(kinds.size(), s);
    p.dk.upload(kinds.data(), kinds.size());
    return p;
}

template <int LPE>
void run_exact(const u64* m, const u64* dec, const std::vector<ExSeg>& segs, const std::vector<ExKind>& kinds,
               ExOut* dout, cudaStream_t s) {
    constexpr u64 C = 32ull * LPE;
    HostTrace ht_prep("exact: prepare");
    Prepared p = prepare(segs, kinds, C, s);
    ht_prep.stop();
    HostTrace ht_launch("exact: launch");
    const int nseg = static_cast<int>(segs.size()), nk = static_cast<int>(kinds.size());
    const int njobs = nseg * nk;
    // short segments: the warp resolves them directly (no tables)
    const bool tables = p.maxlen >= 8 * C;
    DevBuf<double> A, P;
    DevBuf<ExRec> recs;
    if (tables) {
        A = DevBuf<double>(p.nch * nk, s);
        P = DevBuf<double>(p.nch * nk, s);
        recs = DevBuf<ExRec>(p.nch * nk, s);
        const unsigned grid = cdiv(p.nch * nk, kExWarps);
        ex_approx_kernel<LPE><<<grid, 32 * kExWarps, 0, s>>>(m, dec, p.segs.p, nseg, p.dch.p, p.dk.p, nk, p.nch, A.p);
        ex_scan_kernel<<<static_cast<unsigned>(njobs), 1024, 0, s>>>(p.segs.p, nseg, p.dch.p, p.nch, A.p, P.p);
        ex_fn_kernel<LPE><<<grid, 32 * kExWarps, 0, s>>>(m, dec, p.segs.p, nseg, p.dch.p, p.dk.p, nk, p.nch, P.p,
                                                         recs.p);
        count_launch(3);
        TCB_LAUNCH();
    }
    ex_walk_kernel<LPE><<<cdiv(static_cast<u64>(njobs) * 32, 128), 128, 0, s>>>(
        m, dec, p.segs.p, nseg, p.dch.p, p.dk.p, njobs, p.nch, tables ? recs.p : nullptr, dout);
    count_launch();
    TCB_LAUNCH();
}

}  // namespace

struct PlaneStatsJob::Impl {
    const u64* m = nullptr;
    u64 n = 0, block = 0, nb = 0;
    int p_top = 0, np = 0;
    bool generic = false;
    std::vector<ExSeg> segs;
    std::vector<ExKind> kinds;
    Prepared prep;
    DevBuf<double> A, P;
};

PlaneStatsJob::PlaneStatsJob(const u64* m, u64 n, u64 block, int p_top, int np, cudaStream_t s, u64 b0, u64 b1)
    : impl_(std::make_unique<Impl>()), s_(s) {
    if (np < 1 || np > 32 || p_top - np + 1 < 0) throw Error("exact sums: bad plane range");
    Impl& J = *impl_;
    J.m = m;
    J.n = n;
    J.block = block;
    J.p_top = p_top;
    J.np = np;
    const u64 nball = n == 0 ? 0 : (n + block - 1) / block;
    b1 = std::min(b1, nball);
    b0 = std::min(b0, b1);
    J.nb = b1 - b0;
    J.segs.resize(J.nb);
    for (u64 b = b0; b < b1; ++b)
        J.segs[b - b0] = ExSeg{b * block, std::min(n, (b + 1) * block), 0, 0.0, HUGE_VAL};
    for (int l = 0; l < np; ++l) {
        J.kinds.push_back({kExLead, p_top - l});
        J.kinds.push_back({kExTrail, p_top - l});
    }
    static const bool ref_chain = [] {
        const char* e = std::getenv("TCB_EXACT_REFERENCE");
        return e && *e && *e != '0';
    }();
    u64 maxlen = 0;
    for (const auto& g : J.segs) maxlen = std::max(maxlen, g.hi - g.lo);
    // small cores: the generic path (direct warp resolution, no tables)
    J.generic = ref_chain || J.nb == 0 || maxlen < 8 * 2048;
    if (J.generic) return;
    J.prep = prepare(J.segs, J.kinds, 2048, s);
}

PlaneStatsJob::~PlaneStatsJob() = default;

std::vector<double> PlaneStatsJob::approx_residuals() {
    Impl& J = *impl_;
    std::vector<double> t(J.np, 0.0);
    if (J.nb == 0) return t;
    const u64 lo = J.segs.front().lo, hi = J.segs.back().hi;
    const u64 nrun = (hi - lo + kResRun - 1) / kResRun;
    const u64 nsamp_runs = (nrun + kResStride - 1) / kResStride;
    DevBuf<double> d(J.np, s_);
    d.zero();
    const unsigned grid = static_cast<unsigned>(std::max<u64>(1, std::min<u64>(nsamp_runs, 4 * 148)));
    ex_resid_kernel<<<grid, 256, 0, s_>>>(J.m, lo, hi, J.p_top, J.np, d.p);
    count_launch();
    TCB_LAUNCH();
    d.download(t.data(), J.np);
    stream_sync(s_);
    // elements sampled: every kResStride-th run of kResRun (the last run may be short)
    u64 ns = 0;
    for (u64 r = 0; r < nrun; r += kResStride) ns += std::min(kResRun, hi - lo - r * kResRun);
    const double scale = ns ? static_cast<double>(hi - lo) / static_cast<double>(ns) : 0.0;
    for (auto& v : t) v *= scale;
    return t;
}

std::vector<ExOut> PlaneStatsJob::exact(int np_exact) {
    Impl& J = *impl_;
    np_exact = std::max(1, std::min(np_exact, J.np));
    std::vector<ExKind> kinds(J.kinds.begin(), J.kinds.begin() + 2 * np_exact);
    if (J.generic) return exact_serial(J.m, nullptr, J.segs, kinds, s_);
    ProfScope prof(kStats, s_);
    const int nseg = static_cast<int>(J.nb);
    const int njobs = nseg * 2 * np_exact;
    const u64 nch = J.prep.nch;
    const u64 nk = 2 * static_cast<u64>(np_exact);
    J.A = DevBuf<double>(nch * nk, s_);
    J.P = DevBuf<double>(nch * nk, s_);
    // approximate chunk sums of the planes needed (their scans guess each chunk's region)
    constexpr size_t kPlSmem = 4 * 32 * kPlPad * sizeof(u64);
    TCB_ONCE_PER_DEVICE(cudaFuncSetAttribute(ex_plane_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kPlSmem));
                        cudaFuncSetAttribute(ex_plane_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kPlSmem)));
    ex_plane_kernel<0><<<cdiv(nch * 32, 128), 128, kPlSmem, s_>>>(J.m, J.prep.segs.p, nseg, J.prep.dch.p, J.p_top,
                                                                  np_exact, nch, J.A.p, nullptr, nullptr);
    ex_scan_kernel<<<static_cast<unsigned>(njobs), 1024, 0, s_>>>(J.prep.segs.p, nseg, J.prep.dch.p, nch, J.A.p, J.P.p);
    DevBuf<ExRec> recs(nch * 2 * np_exact, s_);
    ex_plane_kernel<1><<<cdiv(nch * 32, 128), 128, kPlSmem, s_>>>(J.m, J.prep.segs.p, nseg, J.prep.dch.p, J.p_top,
                                                                  np_exact, nch, nullptr, J.P.p, recs.p);
    DevBuf<ExOut> d(njobs, s_);
    ex_walk_kernel<64><<<cdiv(static_cast<u64>(njobs) * 32, 128), 128, 0, s_>>>(
        J.m, nullptr, J.prep.segs.p, nseg, J.prep.dch.p, J.prep.dk.p, njobs, nch, recs.p, d.p);
    count_launch(3);
    TCB_LAUNCH();
    std::vector<ExOut> out(njobs);
    d.download(out.data(), njobs);
    stream_sync(s_);
    return out;
}

std::vector<ExOut> exact_plane_stats(const u64* m, u64 n, u64 block, int p_top, int np, cudaStream_t s) {
    PlaneStatsJob job(m, n, block, p_top, np, s);
    return job.exact(np);
}

std::vector<ExOut> exact_serial(const u64* m, const u64* dec, const std::vector<ExSeg>& segs,
                                const std::vector<ExKind>& kinds, cudaStream_t s) {
    static const bool ref_chain = [] {
        const char* e = std::getenv("TCB_EXACT_REFERENCE");
        return e && *e && *e != '0';
    }();
    if (ref_chain) return exact_serial_reference(m, dec, segs, kinds, s);
    ProfScope prof(kSum, s);
    const std::size_t njobs = segs.size() * kinds.size();
    std::vector<ExOut> out(njobs);
    if (njobs == 0) return out;
    DevBuf<ExOut> d(njobs, s);
    u64 maxlen = 0;
    for (const auto& g : segs) maxlen = std::max(maxlen, g.hi - g.lo);
    // few huge sums (the whole-core backward sums): longer chunks, a shorter walk
    if (njobs <= 4 && maxlen >= (u64{1} << 24))
        run_exact<256>(m, dec, segs, kinds, d.p, s);
    else
        run_exact<64>(m, dec, segs, kinds, d.p, s);
    d.download(out.data(), njobs);
    stream_sync(s);
    return out;
}

std::vector<ExOut> exact_serial_reference(const u64* m, const u64* dec, const std::vector<ExSeg>& segs,
                                          const std::vector<ExKind>& kinds, cudaStream_t s) {
    const std::size_t njobs = segs.size() * kinds.size();
    std::vector<ExOut> out(njobs);
    if (njobs == 0) return out;
    Prepared p = prepare(segs, kinds, 2048, s);
    DevBuf<ExOut> d(njobs, s);
    ex_serial_kernel<<<cdiv(njobs, 64), 64, 0, s>>>(m, dec, p.segs.p, static_cast<int>(segs.size()), p.dk.p,
                                                    static_cast<int>(njobs), d.p);
    count_launch();
    TCB_LAUNCH();
    d.download(out.data(), njobs);
    stream_sync(s);
    return out;
}

}  // namespace tcb
