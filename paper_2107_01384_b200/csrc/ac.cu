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
constexpr u32 kSmemEntries = 4096;   // model entries kept in shared memory
constexpr int kBT = 256, kBPer = 8;  // byte pass: 2048 output bytes per CTA
constexpr u64 kBChunk = static_cast<u64>(kBT) * kBPer;

struct JobDev {
    u64 sym_off, out_off, w_off, gws_off;
    u32 cap, hbits;
};

__device__ __forceinline__ u32 hslot(u64 v, u32 hb) {
    return static_cast<u32>((v * 0x9E3779B97F4A7C15ull) >> (64 - hb));
}

// u32 words of one model: hkey (2H) | hval (H) | hpos (H) | cnt (cap) | pre (cap + 1)
__host__ __device__ inline u64 model_words(u32 cap, u32 hbits) { return 4ull * (1ull << hbits) + 2ull * cap + 2; }

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
__global__ void __launch_bounds__(kMT) ac_model_kernel(const u64* __restrict__ syms, const u64* __restrict__ counts,
                                                       int stride, const JobDev* __restrict__ jobs, int njobs,
                                                       const int* __restrict__ ids, u64* __restrict__ recs,
                                                       u32* __restrict__ gws, u32 smem_cap) {
    extern __shared__ __align__(16) u8 am_smem[];
    __shared__ int si[kMT];
    __shared__ u32 red[kMT / 32];
    __shared__ u32 sh_nsym, sh_total, sh_lastesc;
    const int jid = ids ? ids[blockIdx.x] : static_cast<int>(blockIdx.x);
    if (jid >= njobs) return;
    const JobDev jb = jobs[jid];
    const u64 ns = counts[static_cast<u64>(jid) * stride];
    if (ns == 0) return;
    const u32 H = 1u << jb.hbits, hmask = H - 1;
    u32* base = jb.cap <= smem_cap ? reinterpret_cast<u32*>(am_smem) : gws + jb.gws_off;
    u64* hkey = reinterpret_cast<u64*>(base);
    u32* hval = base + 2 * H;
    u32* hpos = hval + H;
    u32* cnt = hpos + H;
    u32* pre = cnt + jb.cap;
    const int t = threadIdx.x;
    for (u32 i = t; i < H; i += kMT) {
        hkey[i] = kEmpty;
        hval[i] = 0;
        hpos[i] = 0xFFFFFFFFu;
    }
    for (u32 i = t; i < jb.cap; i += kMT) cnt[i] = 0;
    __syncthreads();
    if (t == 0) {
        cnt[0] = 1;  // the escape
        pre[0] = 0;
        pre[1] = 1;
        sh_nsym = 1;
        sh_total = 1;
    }
    __syncthreads();
    u64* rc = recs + jb.sym_off;
    const u64* sy = syms + jb.sym_off;
    for (u64 k = 0; k < ns;) {
        const u32 nsym = sh_nsym, total = sh_total;
        // the first symbol whose update finds total + 32 >= 2^16 is coded, then
        // the model halves, then its own increment is applied
        const u32 d = total >= 65504u ? 0u : (65504u - total + 31u) / 32u;
        u32 L = static_cast<u32>(min(static_cast<u64>(kMT), ns - k));
        bool halv = false;
        if (d < L) {
            L = d + 1;
            halv = true;
        }
        const bool act = static_cast<u32>(t) < L;
        u64 v = 0;
        int I = -1;
        u32 slot = 0;
        if (act) {
            v = sy[k + t];
            u32 h = hslot(v, jb.hbits);
            while (true) {
                const u64 key = hkey[h];
                if (key == v) {
                    I = static_cast<int>(hval[h]) - 1;
                    break;
                }
                if (key == kEmpty) break;
                h = (h + 1) & hmask;
            }
        }
        __syncthreads();  // every lookup before any claim
        const bool claim = act && I < 0;
        if (claim) {
            u32 h = hslot(v, jb.hbits);
            while (true) {
                const u64 key = hkey[h];
                if (key == v) break;
                if (key == kEmpty) {
                    const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(&hkey[h]),
                                               static_cast<unsigned long long>(kEmpty),
                                               static_cast<unsigned long long>(v));
                    if (prev == kEmpty || prev == v) break;
                    continue;
                }
                h = (h + 1) & hmask;
            }
            slot = h;
            atomicMin(&hpos[h], static_cast<u32>(t));
        }
        __syncthreads();
        // new values take indices in order of their first occurrence
        const u32 first = (claim && hpos[slot] == static_cast<u32>(t)) ? 1u : 0u;
        u32 nnew;
        const u32 rank = block_excl_scan<kMT>(first, red, nnew);
        if (first) hval[slot] = nsym + rank + 1;
        __syncthreads();
        bool esc = false;
        if (claim) {
            I = static_cast<int>(hval[slot]) - 1;
            esc = first != 0;
        }
        si[t] = act ? I : 0x7fffffff;
        if (act && static_cast<u32>(t) == L - 1) sh_lastesc = esc ? 1u : 0u;
        __syncthreads();
        if (act) {
            // counts at this symbol: chunk-start count + 32 per earlier occurrence
            u32 less = 0, same = 0;
            for (int j = 0; j < t; ++j) {
                const int Ij = si[j];
                less += Ij < I ? 1u : 0u;
                same += Ij == I ? 1u : 0u;
            }
            const u32 T = total + 32u * static_cast<u32>(t);
            u64 rec;
            if (esc) {
                rec = (u64{1} << 32) | (u64{1} << 16) | T;  // escape interval: cum 0, freq 1
            } else {
                const bool old = static_cast<u32>(I) < nsym;
                const u32 cum = (old ? pre[I] : total) + 32u * less;
                const u32 f = (old ? cnt[I] : 0u) + 32u * same;
                rec = (static_cast<u64>(cum) << 48) | (static_cast<u64>(f) << 32) | T;
            }
            rc[k + t] = rec;
        }
        __syncthreads();  // every read of cnt / pre / hpos done
        if (act) {
            if (claim) hpos[slot] = 0xFFFFFFFFu;
            if (!(halv && static_cast<u32>(t) == L - 1)) atomicAdd(&cnt[I], 32u);
        }
        __syncthreads();
        const u32 newn = nsym + nnew;
        if (halv) {
            // an inserted halving symbol is pushed after the halving
            const u32 nh = newn - sh_lastesc;
            for (u32 i = t; i < nh; i += kMT) cnt[i] = max(1u, cnt[i] >> 1);
            __syncthreads();
            if (static_cast<u32>(t) == L - 1) cnt[I] += 32u;
            __syncthreads();
        }
        const u32 per = (newn + kMT - 1) / kMT;
        const u32 i0 = min(newn, static_cast<u32>(t) * per), i1 = min(newn, i0 + per);
        u32 loc = 0;
        for (u32 i = i0; i < i1; ++i) loc += cnt[i];
        u32 tot;
        u32 off = block_excl_scan<kMT>(loc, red, tot);
        for (u32 i = i0; i < i1; ++i) {
            pre[i] = off;
            off += cnt[i];
        }
        if (t == 0) {
            pre[newn] = tot;
            sh_nsym = newn;
            sh_total = tot;
        }
        __syncthreads();
        k += L;
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
    for (u64 k0 = 0; k0 < n1; k0 += 32) {
        const u64 rec_c = ld_rec(k0 + 64);
        const u64 mag_b = magic[rec_b & 0xFFFFu];
        const u32 raw_b = ld_raw(k0 + 32, rec_b);
        const u32 L = static_cast<u32>(min(u64{32}, n1 - k0));
        const unsigned escm = __ballot_sync(0xffffffffu, (rec_a >> 16) & 1u);
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
        rec_a = rec_b;
        mag_a = mag_b;
        raw_a = raw_b;
        rec_b = rec_c;
    }
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

// the largest model's shared memory, opted in once per device (concurrent
// callers on worker threads launch with different sizes below it)
void model_smem_attr() {
    static std::mutex mu;
    static std::map<int, bool> done;
    int dev = 0;
    TCB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (done[dev]) return;
    TCB_CUDA(cudaFuncSetAttribute(ac_model_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(model_words(kSmemEntries, hash_bits(kSmemEntries)) * 4)));
    done[dev] = true;
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

void ac_encode(const u64* syms, const u64* counts, int stride, const std::vector<AcJob>& jobs, u8* ent, u64* elen,
               cudaStream_t s) {
    const int nj = static_cast<int>(jobs.size());
    if (nj == 0) return;
    TCB_CUDA(cudaMemsetAsync(elen, 0, nj * sizeof(u64), s));
    std::vector<JobDev> jd(nj);
    std::vector<u64> choff(nj + 1, 0);
    u64 wtot = 0, gtot = 0, rec_ext = 0;
    std::vector<int> big;
    for (int j = 0; j < nj; ++j) {
        const AcJob& a = jobs[j];
        JobDev& d = jd[j];
        d.sym_off = a.sym_off;
        d.out_off = a.out_off;
        const u64 esc = ac_escape_bound(a.sym_cap, a.positions);
        d.cap = static_cast<u32>(esc + 1);
        d.hbits = hash_bits(d.cap);
        d.w_off = wtot;
        const u64 wcap = a.sym_cap ? 2 * a.sym_cap + 5 * esc + 8 : 0;
        wtot += wcap;
        choff[j + 1] = choff[j] + (wcap + kBChunk - 1) / kBChunk;
        rec_ext = std::max(rec_ext, a.sym_off + a.sym_cap);
        if (d.cap <= kSmemEntries) {
            d.gws_off = 0;
        } else {
            d.gws_off = gtot;
            gtot += (model_words(d.cap, d.hbits) + 3) & ~u64{3};
            big.push_back(j);
        }
    }
    // models of one launch share the dynamic shared-memory size: small ones (most
    // planes) in their own launch so several fit per SM
    DevBuf<JobDev> djobs(nj, s);
    djobs.upload(jd.data(), nj);
    DevBuf<u64> recs(rec_ext + 1, s), W(wtot + 1, s), nout(nj, s), dch(nj + 1, s);
    DevBuf<u32> gws(gtot + 4, s);
    dch.upload(choff.data(), nj + 1);
    const u64 nchunk = choff.back();
    DevBuf<u8> csum(nchunk + 1, s), cin(nchunk + 1, s);
    const u64* magic = magic_table(s);
    {
        ProfScope pa(kAc, s);
        constexpr u32 kSmall = 512;
        std::vector<int> small_ids, large_ids;
        for (int j = 0; j < nj; ++j) (jd[j].cap <= kSmall ? small_ids : large_ids).push_back(j);
        auto launch = [&](const std::vector<int>& ids) {
            if (ids.empty()) return;
            // shared memory for the largest model of this launch that fits; larger
            // models live in their global workspace
            u32 mc = 0;
            for (int j : ids)
                if (jd[j].cap <= kSmemEntries) mc = std::max(mc, jd[j].cap);
            const u64 sm = mc ? model_words(mc, hash_bits(mc)) * 4 : 0;
            model_smem_attr();
            DevBuf<int> dids(ids.size(), s);
            dids.upload(ids.data(), ids.size());
            ac_model_kernel<<<static_cast<unsigned>(ids.size()), kMT, sm, s>>>(syms, counts, stride, djobs.p, nj,
                                                                               dids.p, recs.p, gws.p, mc);
            count_launch();
            TCB_LAUNCH();
        };
        launch(small_ids);
        launch(large_ids);
        ac_range_kernel<<<cdiv(static_cast<u64>(nj) * 32, 128), 128, 0, s>>>(syms, counts, stride, djobs.p, nj, recs.p,
                                                                             magic, W.p, nout.p);
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
}

}  // namespace tcb
