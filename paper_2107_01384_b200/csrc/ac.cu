// Adaptive range coder (entropy.cpp:85-239), bit-exact, in three passes; see
// ac.cuh.  Reference semantics reproduced:
//   RangeEncoder::encode / shift_low / flush   entropy.cpp:85-118
//   AdaptiveModel (escape = index 0 with count 1, +32 per hit, insert with
//   count 32, halve when total + 32 >= 2^16 before bump/insert, escapes carry
//   32 raw bits through encode(bit, 1, 2))     entropy.cpp:155-239
//   encode_symbols framing u8 coder || u32 count || body   entropy.cpp:429-445
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>

#include "ac.cuh"

namespace tcb {

namespace {

constexpr u64 kEmpty = ~u64{0};
constexpr int kMT = 256;             // model threads = symbols per sub-chunk
constexpr int kBT = 256, kBPer = 8;  // byte pass: 2048 output bytes per CTA
constexpr u64 kBChunk = static_cast<u64>(kBT) * kBPer;

struct JobDev {
    u64 sym_off, out_off, w_off, gws_off;
    u64 fp_off, ep_off, snap_off;
    u32 cap, hbits, ep_cap, pad;
};

__device__ __forceinline__ u32 hslot(u64 v, u32 hb) {
    return static_cast<u32>((v * 0x9E3779B97F4A7C15ull) >> (64 - hb));
}


template <int NT>
__device__ __forceinline__ u32 block_excl_scan(u32 v, u32* red, u32& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u32 x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) red[w] = x;
    __syncthreads();
    if (w == 0) {
        u32 z = lane < NT / 32 ? red[lane] : 0u;
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        if (lane < NT / 32) red[lane] = z;  // inclusive
    }
    __syncthreads();
    const u32 before = w > 0 ? red[w - 1] : 0u;
    total = red[NT / 32 - 1];
    __syncthreads();
    return before + x - v;
}

// ---------------------------------------------------------------- 1. model
// Per symbol record: bits 0-15 total, bit 16 escape, 32-47 freq, 48-63 cum.
//
// The adaptive model in three passes:
//  1a. index: a symbol's model index is 1 + the rank of its value's first
//      occurrence (escape = 0), so every symbol is indexed in parallel (hash of
//      values with the minimum position, the distinct values sorted by it);
//  1b. epochs: the only sequential part -- between two halvings every count is
//      its epoch-start value plus 32 per occurrence, so one CTA walks the
//      stream an epoch at a time (a histogram, the halving, the new total) and
//      records each epoch's start counts;
//  1c. code: every epoch of every stream at once, one CTA each: (cum, freq,
//      total) of a symbol = the epoch-start prefix/count plus 32 per earlier
//      occurrence inside the epoch (256-symbol sub-chunks: dominance counts,
//      then a prefix rebuild).
constexpr int kIxT = 1024;  // index / epoch passes
constexpr u32 kIxSmemEntries = 4096;

// u32 words of the index pass's tables: hkey (2H) | hpos (H) | hval (H) | list (2 cap u64:
// the bitonic sort pads the distinct values to a power of two)
__host__ __device__ inline u64 index_words(u32 cap, u32 hbits) { return 4ull * (1ull << hbits) + 4ull * cap; }

__global__ void __launch_bounds__(kIxT) ac_index_kernel(const u64* __restrict__ syms, const u64* __restrict__ counts,
                                                        int stride, const JobDev* __restrict__ jobs, int njobs,
                                                        const int* __restrict__ ids, u32* __restrict__ idx,
                                                        u32* __restrict__ fp, u32* __restrict__ ndist,
                                                        u32* __restrict__ gws, u32 smem_cap, int* __restrict__ err) {
    extern __shared__ __align__(16) u8 ax_smem[];
    __shared__ u32 nd_s;
    const int jid = ids ? ids[blockIdx.x] : static_cast<int>(blockIdx.x);
    if (jid >= njobs) return;
    const JobDev jb = jobs[jid];
    const u64 ns = counts[static_cast<u64>(jid) * stride];
    if (ns == 0) {
        if (threadIdx.x == 0) ndist[jid] = 0;
        return;
    }
    const u32 H = 1u << jb.hbits, hmask = H - 1;
    u32* base = jb.cap <= smem_cap ? reinterpret_cast<u32*>(ax_smem) : gws + jb.gws_off;
    u64* hkey = reinterpret_cast<u64*>(base);
    u32* hpos = base + 2 * H;
    u32* hval = hpos + H;
    u64* list = reinterpret_cast<u64*>(hval + H);
    const u64* sy = syms + jb.sym_off;
    for (u32 i = threadIdx.x; i < H; i += kIxT) {
        hkey[i] = kEmpty;
        hpos[i] = 0xFFFFFFFFu;
    }
    if (threadIdx.x == 0) nd_s = 0;
    __syncthreads();
    for (u64 k = threadIdx.x; k < ns; k += kIxT) {
        const u64 v = sy[k];
        u32 h = hslot(v, jb.hbits);
        while (true) {
            const u64 key = hkey[h];
            if (key == v) break;
            if (key == kEmpty) {
                const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(&hkey[h]),
                                           static_cast<unsigned long long>(kEmpty), static_cast<unsigned long long>(v));
                if (prev == kEmpty || prev == v) break;
                continue;
            }
            h = (h + 1) & hmask;
        }
        atomicMin(&hpos[h], static_cast<u32>(k));
    }
    __syncthreads();
    // the distinct values (position, slot), then sorted by position
    for (u32 i = threadIdx.x; i < H; i += kIxT)
        if (hkey[i] != kEmpty) {
            const u32 at = atomicAdd(&nd_s, 1u);  // index 0 is the escape: at most cap - 1 values
            if (at + 1 < jb.cap) list[at] = (static_cast<u64>(hpos[i]) << 32) | i;
            else *err = 1;
        }
    __syncthreads();
    const u32 D = min(nd_s, jb.cap - 1);
    u32 P2 = 1;
    while (P2 < D) P2 <<= 1;
    for (u32 i = D + threadIdx.x; i < P2; i += kIxT) list[i] = ~u64{0};  // list holds 2 cap >= P2 entries
    __syncthreads();
    for (u32 k = 2; k <= P2; k <<= 1)
        for (u32 j = k >> 1; j > 0; j >>= 1) {
            for (u32 i = threadIdx.x; i < P2; i += kIxT) {
                const u32 l = i ^ j;
                if (l > i) {
                    const u64 a = list[i], b = list[l];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        list[i] = b;
                        list[l] = a;
                    }
                }
            }
            __syncthreads();
        }
    u32* fpj = fp + jb.fp_off;
    for (u32 r = threadIdx.x; r < D; r += kIxT) {
        hval[static_cast<u32>(list[r])] = r + 1;
        fpj[r] = static_cast<u32>(list[r] >> 32);
    }
    if (threadIdx.x == 0) ndist[jid] = D;
    __syncthreads();
    u32* ij = idx + jb.sym_off;
    for (u64 k = threadIdx.x; k < ns; k += kIxT) {
        const u64 v = sy[k];
        u32 h = hslot(v, jb.hbits);
        while (hkey[h] != v) h = (h + 1) & hmask;
        ij[k] = hval[h];
    }
}

// epoch records: (first symbol, total, model size) per epoch; counts snapshot u16 x cap
__global__ void __launch_bounds__(kIxT) ac_epoch_kernel(const u64* __restrict__ counts, int stride,
                                                        const JobDev* __restrict__ jobs, int njobs,
                                                        const u32* __restrict__ idx, const u32* __restrict__ fp,
                                                        const u32* __restrict__ ndist, uint4* __restrict__ eprec,
                                                        u16* __restrict__ snap, u32* __restrict__ nep,
                                                        int* __restrict__ err) {
    extern __shared__ __align__(16) u32 ep_cnt[];
    __shared__ u32 red[kIxT / 32];
    __shared__ u32 sh_nh, sh_nsym;
    const int jid = static_cast<int>(blockIdx.x);
    if (jid >= njobs) return;
    const JobDev jb = jobs[jid];
    const u64 ns = counts[static_cast<u64>(jid) * stride];
    if (ns == 0) {
        if (threadIdx.x == 0) nep[jid] = 0;
        return;
    }
    const u32 cap = jb.cap, D = ndist[jid];
    const u32* ij = idx + jb.sym_off;
    const u32* fpj = fp + jb.fp_off;
    uint4* er = eprec + jb.ep_off;
    u16* sn = snap + jb.snap_off;
    for (u32 i = threadIdx.x; i < cap; i += kIxT) ep_cnt[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) ep_cnt[0] = 1;
    __syncthreads();
    u32 total = 1, nsym = 1, e = 0;
    // number of distinct values whose first occurrence is before position k
    auto first_before = [&](u64 k) {
        u32 lo = 0, hi = D;
        while (lo < hi) {
            const u32 mid = (lo + hi) >> 1;
            if (fpj[mid] < k) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    for (u64 k0 = 0; k0 < ns;) {
        if (e >= jb.ep_cap) {
            if (threadIdx.x == 0) *err = 2;
            break;
        }
        const u32 d = total >= 65504u ? 0u : (65504u - total + 31u) / 32u;
        const u64 kh = k0 + d;
        const bool halv = kh < ns;
        const u64 kend = halv ? kh : ns;
        if (threadIdx.x == 0) er[e] = make_uint4(static_cast<u32>(k0), total, nsym, 0);
        for (u32 i = threadIdx.x; i < nsym; i += kIxT) sn[static_cast<u64>(e) * cap + i] = static_cast<u16>(ep_cnt[i]);
        __syncthreads();
        for (u64 j = k0 + threadIdx.x; j < kend; j += kIxT) atomicAdd(&ep_cnt[ij[j]], 32u);
        ++e;
        if (!halv) break;
        if (threadIdx.x == 0) {
            sh_nh = 1 + first_before(kh);        // the model before the halving symbol's insert
            sh_nsym = 1 + first_before(kh + 1);  // after it
        }
        __syncthreads();
        const u32 nh = sh_nh;
        nsym = sh_nsym;
        for (u32 i = threadIdx.x; i < nh; i += kIxT) ep_cnt[i] = max(1u, ep_cnt[i] >> 1);
        __syncthreads();
        if (threadIdx.x == 0) ep_cnt[ij[kh]] += 32u;
        __syncthreads();
        u32 loc = 0;
        for (u32 i = threadIdx.x; i < nsym; i += kIxT) loc += ep_cnt[i];
        u32 tot;
        block_excl_scan<kIxT>(loc, red, tot);
        total = tot;
        k0 = kh + 1;
    }
    if (threadIdx.x == 0) nep[jid] = e;
}

__device__ __forceinline__ int job_of_slot(const u64* __restrict__ off, int njobs, u64 slot) {
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= slot) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(kMT) ac_code_kernel(const u64* __restrict__ counts, int stride,
                                                      const JobDev* __restrict__ jobs, int njobs,
                                                      const u64* __restrict__ epslot, const u32* __restrict__ idx,
                                                      const u32* __restrict__ fp, const u32* __restrict__ ndist,
                                                      const uint4* __restrict__ eprec, const u16* __restrict__ snap,
                                                      const u32* __restrict__ nep, u64* __restrict__ recs) {
    extern __shared__ __align__(16) u32 cd_smem[];
    __shared__ int si[kMT];
    __shared__ u32 red[kMT / 32];
    const u64 slot = blockIdx.x;
    const int jid = job_of_slot(epslot, njobs, slot);
    const u32 e = static_cast<u32>(slot - epslot[jid]);
    const u32 ne = nep[jid];
    if (e >= ne) return;
    const JobDev jb = jobs[jid];
    const u64 ns = counts[static_cast<u64>(jid) * stride];
    const uint4 r0 = eprec[jb.ep_off + e];
    const u64 k0 = r0.x, k1 = e + 1 < ne ? eprec[jb.ep_off + e + 1].x : ns;
    const u32 T0 = r0.y, nsym0 = r0.z;
    const u32 nend = e + 1 < ne ? eprec[jb.ep_off + e + 1].z : ndist[jid] + 1;  // model size at the epoch end
    u32* cnt = cd_smem;
    u32* pre = cnt + jb.cap;
    const u16* sn = snap + jb.snap_off + static_cast<u64>(e) * jb.cap;
    const u32* ij = idx + jb.sym_off;
    const u32* fpj = fp + jb.fp_off;
    u64* rc = recs + jb.sym_off;
    const int t = threadIdx.x;
    for (u32 i = t; i < nend; i += kMT) cnt[i] = i < nsym0 ? sn[i] : 0u;
    __syncthreads();
    auto rebuild_prefix = [&]() {
        const u32 per = (nend + kMT - 1) / kMT;
        const u32 i0 = min(nend, static_cast<u32>(t) * per), i1 = min(nend, i0 + per);
        u32 loc = 0;
        for (u32 i = i0; i < i1; ++i) loc += cnt[i];
        u32 tot;
        u32 off = block_excl_scan<kMT>(loc, red, tot);
        for (u32 i = i0; i < i1; ++i) {
            pre[i] = off;
            off += cnt[i];
        }
        __syncthreads();
    };
    rebuild_prefix();
    for (u64 k = k0; k < k1; k += kMT) {
        const u64 kk = k + t;
        const bool act = kk < k1;
        const int I = act ? static_cast<int>(ij[kk]) : 0x7fffffff;
        si[t] = I;
        __syncthreads();
        if (act) {
            u32 less = 0, same = 0;
            for (int j = 0; j < t; ++j) {
                const int Ij = si[j];
                less += Ij < I ? 1u : 0u;
                same += Ij == I ? 1u : 0u;
            }
            const u32 T = T0 + 32u * static_cast<u32>(kk - k0);
            u64 rec;
            if (I == 0 || fpj[I - 1] == static_cast<u32>(kk)) {  // (I == 0 only after a capacity error)
                rec = (u64{1} << 32) | (u64{1} << 16) | T;  // escape: cum 0, freq 1
            } else {
                const u32 cum = pre[I] + 32u * less;
                const u32 f = cnt[I] + 32u * same;
                rec = (static_cast<u64>(cum) << 48) | (static_cast<u64>(f) << 32) | T;
            }
            rc[kk] = rec;
        }
        __syncthreads();
        if (act) atomicAdd(&cnt[I], 32u);
        __syncthreads();
        if (k + kMT < k1) rebuild_prefix();
    }
}

// ---------------------------------------------------------------- 2. range recurrence
// One warp per stream; lanes hold 32 consecutive records (loaded two chunks
// ahead, their divisor reciprocals one chunk ahead) and every lane runs the
// identical recurrence.  floor(range / T) = (range * M_hi + umulhi(range,
// M_lo)) >> 32 with M = ceil(2^64 / T): exact for range < 2^32, 1 < T < 2^16.
__global__ void __launch_bounds__(128) ac_range_kernel(const u64* __restrict__ syms, const u64* __restrict__ counts,
                                                       int stride, const JobDev* __restrict__ jobs, int njobs,
                                                       const u64* __restrict__ recs, const u64* __restrict__ magic,
                                                       u64* __restrict__ W, u64* __restrict__ nout) {
    const int j = static_cast<int>((static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    if (j >= njobs) return;
    const int lane = threadIdx.x & 31;
    __shared__ ulonglong2 stage[4][32];
    __shared__ uint4 stage4[4][32];
    __shared__ u32 rin_sh[2][4][32];
    const int wib = threadIdx.x >> 5;
    const JobDev jb = jobs[j];
    const u64 ns = counts[static_cast<u64>(j) * stride];
    if (ns == 0) {
        if (lane == 0) nout[j] = 0;
        return;
    }
    const u64* sy = syms + jb.sym_off;
    u64* const w0 = W + jb.w_off;
    u64* w = w0;  // W[S]: running pointer (S = w - w0)
    const bool l0 = lane == 0;
    u32 range = 0xFFFFFFFFu;
    u64 acc = 0;
    // 32 raw bits, MSB first, each encode(bit, 1, 2): with range in [2^24, 2^32)
    // exactly floor(log2 range) - 23 halvings fit before a normalisation, so the
    // bits go in groups: low += sum_j bit_j (range >> j), range >>= k
    auto raw_bits = [&](u32 raw) {
        int left = 32;
        while (left > 0) {
            const int kb = min(left, (31 - __clz(static_cast<int>(range))) - 23);
            const u32 cb = (raw >> (left - kb)) & ((1u << kb) - 1u);
            u64 add = 0;
#pragma unroll
            for (int jj = 1; jj <= 8; ++jj)
                if (jj <= kb && ((cb >> (kb - jj)) & 1u)) add += range >> jj;
            acc += add;
            range >>= kb;
            left -= kb;
            while (range < (1u << 24)) {
                if (l0) *w = acc;
                ++w;
                acc = 0;
                range <<= 8;
            }
        }
    };
    // the first symbol is always an escape against total 1: range / 1, cum 0, freq 1
    raw_bits(static_cast<u32>(sy[0]));
    // symbols 1.. : total >= 2 from here on
    const u64* rc = recs + jb.sym_off + 1;
    const u64* sy1 = sy + 1;
    const u64 n1 = ns - 1;
    auto ld_rec = [&](u64 k0) { return k0 + lane < n1 ? rc[k0 + lane] : u64{0}; };
    auto ld_raw = [&](u64 k0, u64 rec) { return ((rec >> 16) & 1u) ? static_cast<u32>(sy1[k0 + lane]) : 0u; };
    // one coding step: q = floor(range / T) by multiply-high with M = ceil(2^64 / T)
    // (exact for range < 2^32, 1 < T < 2^16); q >= 2^8, so at most two shifts
    auto step = [&](u64 rec, u64 M) {
        const u32 hi = static_cast<u32>(rec >> 32);
        const u32 t = __umulhi(range, static_cast<u32>(M));
        const u32 q = static_cast<u32>((static_cast<u64>(range) * static_cast<u32>(M >> 32) + t) >> 32);
        acc += static_cast<u64>(hi >> 16) * q;
        const u32 rr = q * (hi & 0xFFFFu);
        // every lane stores the running slot (identical values): the last store to
        // a slot is its complete sum, a skipped slot gets its zero
        w[0] = acc;
        w[1] = 0;
        const u32 r1 = rr < (1u << 24) ? rr << 8 : rr;
        range = r1 < (1u << 24) ? r1 << 8 : r1;
        const u32 sh = (rr < (1u << 24) ? 1u : 0u) + (rr < (1u << 16) ? 1u : 0u);
        w += sh;
        acc = sh ? 0 : acc;
    };
    u64 rec_a = ld_rec(0), rec_b = ld_rec(32);
    u64 mag_a = magic[rec_a & 0xFFFFu];
    u32 raw_a = ld_raw(0, rec_a);
    // Full chunks without escapes run software-pipelined: the range chain of
    // chunk k (32 dependent steps, each step's incoming range kept per lane)
    // sits in one basic block with the parallel part of chunk k - 1 (the
    // additions to `low`, shift counts and slot stores by the 32 lanes), whose
    // independent instructions fill the chain's latency gaps.  A chunk with an
    // escape (or the partial last one) first completes the pending parallel
    // part, then steps serially.
    bool pend = false;          // a chunk's parallel part is pending
    u32 p_rin = 0;              // its lane's incoming range
    u64 p_rec = 0, p_mag = 0;   // its lane's record and reciprocal
    int buf = 0;
    auto finish = [&](u32 rin, u64 rec, u64 mag) {  // the parallel part of one chunk
        const u32 hi = static_cast<u32>(rec >> 32);
        const u32 t = __umulhi(rin, static_cast<u32>(mag));
        const u32 q = static_cast<u32>((static_cast<u64>(rin) * static_cast<u32>(mag >> 32) + t) >> 32);
        const u64 add = static_cast<u64>(hi >> 16) * q;
        const u32 rr = q * (hi & 0xFFFFu);
        const u32 sh = (rr < (1u << 24) ? 1u : 0u) + (rr < (1u << 16) ? 1u : 0u);
        u32 isum = sh;
        u64 iadd = add;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 ys = __shfl_up_sync(0xffffffffu, isum, o);
            const u64 ya = __shfl_up_sync(0xffffffffu, iadd, o);
            if (lane >= o) {
                isum += ys;
                iadd += ya;
            }
        }
        const unsigned smask = __ballot_sync(0xffffffffu, sh != 0);
        const unsigned below = smask & ((1u << lane) - 1u);
        const int prev = below ? 31 - __clz(static_cast<int>(below)) : 0;
        const u64 base = __shfl_sync(0xffffffffu, iadd, prev);
        const int last = smask ? 31 - __clz(static_cast<int>(smask)) : 0;
        const u64 at_last = __shfl_sync(0xffffffffu, iadd, last);
        const u64 tot = __shfl_sync(0xffffffffu, iadd, 31);
        const u32 nsh = __shfl_sync(0xffffffffu, isum, 31);
        if (sh) {  // this step closes slot S0 + pos (its sum: the steps since the previous close)
            const u32 pos = isum - sh;
            w[pos] = below ? iadd - base : acc + iadd;
            if (sh == 2) w[pos + 1] = 0;
        }
        acc = smask ? tot - at_last : acc + tot;
        w += nsh;
    };
    for (u64 k0 = 0; k0 < n1; k0 += 32) {
        const u64 rec_c = ld_rec(k0 + 64);
        const u64 mag_b = magic[rec_b & 0xFFFFu];
        const u32 raw_b = ld_raw(k0 + 32, rec_b);
        const u32 L = static_cast<u32>(min(u64{32}, n1 - k0));
        const unsigned escm = __ballot_sync(0xffffffffu, (rec_a >> 16) & 1u);
        if (escm == 0 && L == 32) {
            // per-step 16-byte records: reciprocal, and the normalisation decided
            // from q by thresholds (q f < 2^24 <=> q < ceil(2^24 / f)), so it is a
            // select of the multiplier beside the quotient
            {
                const u32 f = static_cast<u32>(rec_a >> 32) & 0xFFFFu;
                const u32 th1 = ((1u << 24) + f - 1) / f, th2 = ((1u << 16) + f - 1) / f;
                __syncwarp();
                stage4[wib][lane] = make_uint4(static_cast<u32>(mag_a), static_cast<u32>(mag_a >> 32),
                                               f | ((th2 - 1) << 16), th1);
                __syncwarp();
            }
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const uint4 d = stage4[wib][u];
                rin_sh[buf][wib][u] = range;
                const u32 f = d.z & 0xFFFFu;
                const u32 t = __umulhi(range, d.x);
                const u32 q = static_cast<u32>((static_cast<u64>(range) * d.y + t) >> 32);
                const u32 mul = q <= (d.z >> 16) ? f << 16 : (q < d.w ? f << 8 : f);
                range = q * mul;
            }
            if (pend) finish(p_rin, p_rec, p_mag);  // the previous chunk, beside this chain
            __syncwarp();
            p_rin = rin_sh[buf][wib][lane];
            p_rec = rec_a;
            p_mag = mag_a;
            pend = true;
            buf ^= 1;
        } else {
            if (pend) {
                finish(p_rin, p_rec, p_mag);
                pend = false;
            }
            // the chunk's (record, reciprocal) pairs go through shared memory: the
            // steps read them with broadcast loads the compiler issues ahead
            __syncwarp();
            stage[wib][lane] = make_ulonglong2(rec_a, mag_a);
            __syncwarp();
            for (u32 g = 0; g < L; g += 8) {
                const unsigned em = (escm >> g) & 0xFFu;
                if (em == 0 && g + 8 <= L) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const ulonglong2 rm = stage[wib][g + u];
                        step(rm.x, rm.y);
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        if (g + u >= L) break;
                        const ulonglong2 rm = stage[wib][g + u];
                        step(rm.x, rm.y);
                        if ((em >> u) & 1u) raw_bits(__shfl_sync(0xffffffffu, raw_a, g + u));
                    }
                }
            }
        }
        rec_a = rec_b;
        mag_a = mag_b;
        raw_a = raw_b;
        rec_b = rec_c;
    }
    if (pend) finish(p_rin, p_rec, p_mag);
    if (lane == 0) {  // flush: five shift_low calls
        w[0] = acc;
        for (int i = 1; i < 5; ++i) w[i] = 0;
        nout[j] = static_cast<u64>(w - w0) + 5;
    }
}

// ---------------------------------------------------------------- 3. bytes
// Output byte i is digit i of Z = sum_S W[S] 256^(N-5-S): raw digit sum
// R(i) = sum_{b<5} byte_b(W[i-4+b]); V(i) = R(i) mod 256 + R(i+1) div 256;
// then a carry c in {0,1} runs from the last byte to the first.
__device__ __forceinline__ u32 digit_sum(const u64* __restrict__ w, u64 N, long long i) {
    u32 r = 0;
#pragma unroll
    for (int b = 0; b < 5; ++b) {
        const long long s = i - 4 + b;
        if (s >= 0 && static_cast<u64>(s) < N) r += static_cast<u32>((w[s] >> (8 * b)) & 0xFFu);
    }
    return r;
}

// carry function of a run: bit c = carry out for carry in c; identity = 0b10
__device__ __forceinline__ u32 cf_then(u32 f, u32 g) {  // g (right part) first, then f
    return ((f >> (g & 1u)) & 1u) | (((f >> ((g >> 1) & 1u)) & 1u) << 1);
}

__device__ __forceinline__ int chunk_job(const u64* __restrict__ choff, int njobs, u64 c) {
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (choff[mid] <= c) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// this thread's 8 digits (before the carry) and its carry function
__device__ __forceinline__ u32 thread_digits(const u64* __restrict__ w, u64 N, u64 i0, u32 (&V)[kBPer]) {
    u32 R[kBPer + 1];
#pragma unroll
    for (int p = 0; p <= kBPer; ++p) R[p] = i0 + p < N ? digit_sum(w, N, static_cast<long long>(i0 + p)) : 0u;
    u32 f = 2u;
#pragma unroll
    for (int p = kBPer - 1; p >= 0; --p) {
        V[p] = i0 + p < N ? (R[p] & 0xFFu) + (R[p + 1] >> 8) : 0u;
        const u32 c0 = (f & 1u), c1 = (f >> 1) & 1u;  // carry into p for carry-in 0/1
        f = ((V[p] + c0) >> 8 ? 1u : 0u) | (((V[p] + c1) >> 8 ? 1u : 0u) << 1);
    }
    return f;
}

// inclusive suffix composition over the CTA; returns this thread's carry-in function
// (composition of the threads to its right) and the whole CTA's function
__device__ __forceinline__ u32 cta_suffix(u32 f, u32* sh, u32& all) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u32 s = f;
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_down_sync(0xffffffffu, s, o);
        if (lane + o < 32) s = cf_then(s, y);
    }
    u32 ex = __shfl_down_sync(0xffffffffu, s, 1);
    if (lane == 31) ex = 2u;
    if (lane == 0) sh[w] = s;
    __syncthreads();
    u32 right = 2u;  // warps to the right of this one
    for (int q = kBT / 32 - 1; q > w; --q) right = cf_then(sh[q], right);
    all = 2u;
    for (int q = kBT / 32 - 1; q >= 0; --q) all = cf_then(sh[q], all);
    __syncthreads();
    return cf_then(ex, right);
}

__global__ void __launch_bounds__(kBT) ac_bytes_summary(const u64* __restrict__ W, const JobDev* __restrict__ jobs,
                                                        int njobs, const u64* __restrict__ nout,
                                                        const u64* __restrict__ choff, u8* __restrict__ csum) {
    __shared__ u32 sh[kBT / 32];
    const u64 c = blockIdx.x;
    const int j = chunk_job(choff, njobs, c);
    const u64 N = nout[j];
    const u64 base = (c - choff[j]) * kBChunk;
    if (base >= N) return;
    u32 V[kBPer];
    const u32 f = thread_digits(W + jobs[j].w_off, N, base + static_cast<u64>(threadIdx.x) * kBPer, V);
    u32 all;
    cta_suffix(f, sh, all);
    if (threadIdx.x == 0) csum[c] = static_cast<u8>(all);
}

__global__ void ac_bytes_carry(const u64* __restrict__ nout, const u64* __restrict__ choff, int njobs,
                               const u8* __restrict__ csum, u8* __restrict__ cin) {
    const int j = static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x);
    if (j >= njobs) return;
    const u64 nch = (nout[j] + kBChunk - 1) / kBChunk;
    u32 carry = 0;
    for (u64 q = nch; q-- > 0;) {
        cin[choff[j] + q] = static_cast<u8>(carry);
        carry = (csum[choff[j] + q] >> carry) & 1u;
    }
}

__global__ void __launch_bounds__(kBT) ac_bytes_write(const u64* __restrict__ W, const JobDev* __restrict__ jobs,
                                                      int njobs, const u64* __restrict__ nout,
                                                      const u64* __restrict__ counts, int stride,
                                                      const u64* __restrict__ choff, const u8* __restrict__ cin,
                                                      u8* __restrict__ ent, u64* __restrict__ elen) {
    __shared__ u32 sh[kBT / 32];
    const u64 c = blockIdx.x;
    const int j = chunk_job(choff, njobs, c);
    const u64 N = nout[j];
    const u64 base = (c - choff[j]) * kBChunk;
    const JobDev jb = jobs[j];
    u8* out = ent + jb.out_off;
    if (base == 0 && threadIdx.x == 0) {
        if (N == 0) {
            elen[j] = 0;
        } else {
            const u32 n32 = static_cast<u32>(counts[static_cast<u64>(j) * stride]);
            out[0] = 0;  // coder id: arithmetic
            for (int b = 0; b < 4; ++b) out[1 + b] = static_cast<u8>(n32 >> (8 * b));
            elen[j] = 5 + N;
        }
    }
    if (base >= N) return;
    const u64 i0 = base + static_cast<u64>(threadIdx.x) * kBPer;
    u32 V[kBPer];
    const u32 f = thread_digits(W + jb.w_off, N, i0, V);
    u32 all;
    const u32 g = cta_suffix(f, sh, all);
    u32 carry = (g >> cin[c]) & 1u;
#pragma unroll
    for (int p = kBPer - 1; p >= 0; --p) {
        if (i0 + p >= N) continue;
        const u32 x = V[p] + carry;
        out[5 + i0 + p] = static_cast<u8>(x);
        carry = x >> 8;
    }
}

__global__ void magic_kernel(u64* m) {
    const u32 T = blockIdx.x * blockDim.x + threadIdx.x;
    if (T < 65536) m[T] = T > 1 ? (~u64{0} / T) + 1 : 0;
}

const u64* magic_table(cudaStream_t s) {
    static std::mutex mu;
    static std::map<int, u64*> tabs;
    int dev = 0;
    TCB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = tabs.find(dev);
    if (it != tabs.end()) return it->second;
    u64* p = nullptr;
    TCB_CUDA(cudaMalloc(&p, 65536 * sizeof(u64)));
    magic_kernel<<<256, 256, 0, s>>>(p);
    count_launch();
    TCB_LAUNCH();
    TCB_CUDA(cudaStreamSynchronize(s));
    tabs[dev] = p;
    return p;
}

u32 hash_bits(u32 cap);
// Code length bounds without the sequential range pass: the coder shifts out
// S bytes with 24 <= log2(range_end) = log2(range_0) - C - E + 8 S < 32, where
// C = sum log2(T / f) over the symbols (+ 1 per raw escape bit) and E = the
// floor(range / T) truncation losses, each in [0, log2(1 / (1 - T / range)))
// with range >= 2^24, T < 2^16.  Output bytes = 5 (framing) + S + 5 (flush).
__global__ void __launch_bounds__(256) ac_bounds_kernel(const u64* __restrict__ counts, int stride,
                                                        const JobDev* __restrict__ jobs, int njobs,
                                                        const u64* __restrict__ recs, u64* __restrict__ lo_hi) {
    __shared__ double red[2][8];
    const int j = blockIdx.x;
    if (j >= njobs) return;
    const JobDev jb = jobs[j];
    const u64 ns = counts[static_cast<u64>(j) * stride];
    double c = 0.0, e = 0.0;
    const u64* rc = recs + jb.sym_off;
    for (u64 k = threadIdx.x; k < ns; k += blockDim.x) {
        if (k == 0) {  // the first symbol (escape against total 1): 32 raw bits, log2(1) = 0
            c += 32.0;
            e += 32.0 * 1.8e-7;
            continue;
        }
        const u64 r = rc[k];
        const double T = static_cast<double>(r & 0xFFFFu), f = static_cast<double>((r >> 32) & 0xFFFFu);
        c += log2(T) - log2(f);
        e += 0.005646;  // log2(1 / (1 - 2^-8)) rounded up
        if ((r >> 16) & 1u) {
            c += 32.0;
            e += 32.0 * 1.8e-7;  // a raw bit: floor(range / 2), range >= 2^24
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        c += __shfl_xor_sync(0xffffffffu, c, o);
        e += __shfl_xor_sync(0xffffffffu, e, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = c;
        red[1][threadIdx.x >> 5] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double C = 0.0, E = 0.0;
        for (int w = 0; w < 8; ++w) {
            C += red[0][w];
            E += red[1][w];
        }
        if (ns == 0) {
            lo_hi[2 * j] = lo_hi[2 * j + 1] = 0;
            return;
        }
        const double slack = 1e-9 * C + 1e-6;  // rounding of the log sums
        const double smin = ceil((C - slack - 8.0) / 8.0), smax = floor((C + E + slack + 1e-8) / 8.0);
        lo_hi[2 * j] = 10 + static_cast<u64>(max(smin, 0.0));
        lo_hi[2 * j + 1] = 10 + static_cast<u64>(max(smax, 0.0));
    }
}

// the largest index-pass tables, opted in once per device (concurrent callers
// on worker threads launch with different sizes below it)
void model_smem_attr() {
    TCB_ONCE_PER_DEVICE({
        cudaFuncSetAttribute(ac_index_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(index_words(kIxSmemEntries, hash_bits(kIxSmemEntries)) * 4));
        cudaFuncSetAttribute(ac_epoch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(ac_code_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    });
}

u32 hash_bits(u32 cap) {
    u32 b = 5;
    while ((1u << b) < 2 * cap) ++b;
    return b;
}

}  // namespace

u64 ac_escape_bound(u64 sym_cap, u64 positions) {
    const u64 d = static_cast<u64>(std::sqrt(2.0 * static_cast<double>(positions))) + 2;
    return std::min(sym_cap, d);
}

u64 ac_out_cap(u64 sym_cap, u64 positions) {
    if (sym_cap == 0) return 0;
    return 5 + 2 * sym_cap + 5 * ac_escape_bound(sym_cap, positions) + 8;
}

namespace {
void ac_run(const u64* syms, const u64* counts, int stride, const std::vector<AcJob>& jobs, u8* ent, u64* elen,
            u64* bounds, cudaStream_t s, int* err_ext = nullptr, const std::function<void()>* launched = nullptr) {
    const int nj = static_cast<int>(jobs.size());
    if (nj == 0) return;
    if (elen) TCB_CUDA(cudaMemsetAsync(elen, 0, nj * sizeof(u64), s));
    std::vector<JobDev> jd(nj);
    std::vector<u64> choff(nj + 1, 0), epslot(nj + 1, 0);
    u64 wtot = 0, gtot = 0, rec_ext = 0, fptot = 0, eptot = 0, sntot = 0;
    u32 cap_max = 1;
    for (int j = 0; j < nj; ++j) {
        const AcJob& a = jobs[j];
        JobDev& d = jd[j];
        d.sym_off = a.sym_off;
        d.out_off = a.out_off;
        const u64 esc = a.distinct ? std::min(a.sym_cap, a.distinct) : ac_escape_bound(a.sym_cap, a.positions);
        d.cap = static_cast<u32>(esc + 1);
        d.hbits = hash_bits(d.cap);
        cap_max = std::max(cap_max, d.cap);
        d.w_off = wtot;
        const u64 wcap = a.sym_cap ? 2 * a.sym_cap + 5 * esc + 8 : 0;
        wtot += wcap;
        choff[j + 1] = choff[j] + (wcap + kBChunk - 1) / kBChunk;
        rec_ext = std::max(rec_ext, a.sym_off + a.sym_cap);
        d.fp_off = fptot;
        fptot += d.cap;
        // an epoch holds at least (65504 - 32768 - cap - 32) / 32 symbols after the first halving
        const u64 dmin = d.cap < 32000 ? (65504 - 32768 - d.cap - 32) / 32 : 1;
        d.ep_cap = static_cast<u32>(a.sym_cap / std::max<u64>(dmin, 1) + 4);
        d.ep_off = eptot;
        eptot += d.ep_cap;
        epslot[j + 1] = eptot;
        d.snap_off = sntot;
        sntot += static_cast<u64>(d.ep_cap) * d.cap;
        if (d.cap <= kIxSmemEntries) {
            d.gws_off = 0;
        } else {
            d.gws_off = gtot;
            gtot += (index_words(d.cap, d.hbits) + 3) & ~u64{3};
        }
    }
    if (cap_max > 24000) throw Error("entropy: more than 24000 distinct symbols in one stream");
    DevBuf<JobDev> djobs(nj, s);
    djobs.upload(jd.data(), nj);
    DevBuf<u64> recs(rec_ext + 1, s), W(wtot + 1, s), nout(nj, s), dch(nj + 1, s), dep(nj + 1, s);
    DevBuf<u32> gws(gtot + 4, s), idx(rec_ext + 1, s), fp(fptot + 1, s), ndist(nj, s), nep(nj, s);
    DevBuf<uint4> eprec(eptot + 1, s);
    DevBuf<u16> snap(sntot + 1, s);
    DevBuf<int> err_own;
    int* errp = err_ext;
    if (!errp) {
        err_own = DevBuf<int>(1, s);
        err_own.zero();
        errp = err_own.p;
    }
    dch.upload(choff.data(), nj + 1);
    dep.upload(epslot.data(), nj + 1);
    const u64 nchunk = choff.back();
    DevBuf<u8> csum(nchunk + 1, s), cin(nchunk + 1, s);
    const u64* magic = magic_table(s);
    {
        ProfScope pa(kAc, s);
        model_smem_attr();
        constexpr u32 kSmall = 512;
        std::vector<int> small_ids, large_ids;
        for (int j = 0; j < nj; ++j) (jd[j].cap <= kSmall ? small_ids : large_ids).push_back(j);
        for (const auto* ids : {&small_ids, &large_ids}) {  // tables sized per launch: small models pack an SM
            if (ids->empty()) continue;
            u32 mc = 0;
            for (int j : *ids)
                if (jd[j].cap <= kIxSmemEntries) mc = std::max(mc, jd[j].cap);
            const u64 sm = mc ? index_words(mc, hash_bits(mc)) * 4 : 0;
            DevBuf<int> dids(ids->size(), s);
            dids.upload(ids->data(), ids->size());
            ac_index_kernel<<<static_cast<unsigned>(ids->size()), kIxT, sm, s>>>(
                syms, counts, stride, djobs.p, nj, dids.p, idx.p, fp.p, ndist.p, gws.p, mc, errp);
            count_launch();
            TCB_LAUNCH();
        }
        ac_epoch_kernel<<<static_cast<unsigned>(nj), kIxT, cap_max * sizeof(u32), s>>>(
            counts, stride, djobs.p, nj, idx.p, fp.p, ndist.p, eprec.p, snap.p, nep.p, errp);
        ac_code_kernel<<<static_cast<unsigned>(eptot), kMT, 2 * (cap_max + 1) * sizeof(u32), s>>>(
            counts, stride, djobs.p, nj, dep.p, idx.p, fp.p, ndist.p, eprec.p, snap.p, nep.p, recs.p);
        count_launch(2);
        TCB_LAUNCH();
        if (bounds) {  // code-length bounds only: no range recurrence, no bytes
            ac_bounds_kernel<<<static_cast<unsigned>(nj), 256, 0, s>>>(counts, stride, djobs.p, nj, recs.p, bounds);
            count_launch();
            TCB_LAUNCH();
            if (launched && *launched) (*launched)();
            if (err_ext) return;
            int herr = 0;
            d2h(&herr, errp, sizeof(int), s);
            stream_sync(s);
            if (herr) throw Error("entropy: device model capacity exceeded");
            return;
        }
        // Each stream's recurrence is one dependent chain: when the CTAs (4 streams
        // each) fit one per SM, a shared-memory reservation keeps every other
        // kernel's CTAs off their SMs, so each chain has a scheduler to itself
        // (co-resident warps measured ~30 % slower chains on c5).
        const unsigned rgrid = cdiv(static_cast<u64>(nj) * 32, 128);
        const bool exclusive = rgrid <= static_cast<unsigned>(sm_count());
        constexpr int kRangeExclusiveSmem = 215 * 1024;
        if (exclusive)
            TCB_ONCE_PER_DEVICE(cudaFuncSetAttribute(ac_range_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     kRangeExclusiveSmem));
        ac_range_kernel<<<rgrid, 128, exclusive ? kRangeExclusiveSmem : 0, s>>>(syms, counts, stride, djobs.p, nj,
                                                                                recs.p, magic, W.p, nout.p);
        count_launch();
        TCB_LAUNCH();
        if (nchunk) {
            ac_bytes_summary<<<static_cast<unsigned>(nchunk), kBT, 0, s>>>(W.p, djobs.p, nj, nout.p, dch.p, csum.p);
            ac_bytes_carry<<<cdiv(nj, 128), 128, 0, s>>>(nout.p, dch.p, nj, csum.p, cin.p);
        }
        count_launch(2);
        TCB_LAUNCH();
        // every stream's framing and elen (streams without symbols have no chunks)
        ac_bytes_write<<<static_cast<unsigned>(std::max<u64>(nchunk, 1)), kBT, 0, s>>>(
            W.p, djobs.p, nj, nout.p, counts, stride, dch.p, cin.p, ent, elen);
        count_launch();
        TCB_LAUNCH();
    }
    if (err_ext) return;  // the caller reads the flag with its results
    int herr = 0;
    d2h(&herr, errp, sizeof(int), s);
    stream_sync(s);
    if (herr) throw Error("entropy: device model capacity exceeded");
}
}  // namespace

void ac_encode(const u64* syms, const u64* counts, int stride, const std::vector<AcJob>& jobs, u8* ent, u64* elen,
               cudaStream_t s, int* err_dev) {
    ac_run(syms, counts, stride, jobs, ent, elen, nullptr, s, err_dev);
}

std::vector<u64> ac_size_bounds(const u64* syms, const u64* counts, int stride, const std::vector<AcJob>& jobs,
                                cudaStream_t s, const std::function<void()>& launched) {
    const std::size_t nj = jobs.size();
    std::vector<u64> out(2 * nj, 0);
    if (nj == 0) {
        if (launched) launched();
        return out;
    }
    DevBuf<u64> d(2 * nj, s);
    ac_run(syms, counts, stride, jobs, nullptr, nullptr, d.p, s, nullptr, &launched);
    d.download(out.data(), 2 * nj);
    stream_sync(s);
    return out;
}

}  // namespace tcb
