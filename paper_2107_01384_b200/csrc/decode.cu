// Device decode of the container's bit-plane streams (corecodec::decode,
// core_codec.cpp:421-508; entropy decoders entropy.cpp:82-239, 290-421) and
// the dtype emit of pipeline::decompress (container.cpp:98-140).
//
//   dec_entropy_kernel : every (stream, plane, block) entropy section at once,
//                        one warp per section.  Adaptive range decoder with the
//                        model in shared memory (index 0 = escape, +32 per hit,
//                        halving when total + 32 reaches 2^16), symbol lookup by
//                        a warp-parallel 3-level (1024 / 32 / 1) prefix search;
//                        rANS sections are decoded by lane 0 (semi-static table).
//   dec_stream_kernel  : one CTA per (stream, block), planes in order, the
//                        coefficients of a plane in parallel: a coefficient's
//                        leading-column bit is the run-expanded column at its
//                        rank among the still-insignificant coefficients, its raw
//                        bit the one at its rank among the bit consumers
//                        (refinements up to the trail stop, new ones' signs).
//   emit_kernel        : cast_out<Native> (round-to-nearest-even + clamping for
//                        integers, plain conversion for floats).
#include <cmath>
#include <cstdint>
#include <limits>
#include <type_traits>

#include "decode.cuh"
#include "kernels.cuh"

namespace tcb {

namespace {

constexpr u32 kDecCap = 2048;  // model entries in shared memory (global scratch beyond)

__device__ __forceinline__ u32 dec_le32(const u8* p) {
    return static_cast<u32>(p[0]) | (static_cast<u32>(p[1]) << 8) | (static_cast<u32>(p[2]) << 16) |
           (static_cast<u32>(p[3]) << 24);
}

__device__ void dec_fail(int* err, int code) { atomicCAS(err, 0, code); }

// ---------------------------------------------------------------- adaptive range decoder
// Model layout (u32 words): cnt[cap] | l1[cap/32+1] | l2[cap/1024+1] | val[cap] (u64, 8-aligned)
__host__ __device__ inline u64 dec_model_words(u32 cap) {
    const u64 w = cap + (cap / 32 + 1) + (cap / 1024 + 1);
    return ((w + 1) & ~u64{1}) + 2ull * cap;
}

template <bool kShared>
__global__ void __launch_bounds__(32) dec_entropy_kernel(const u8* __restrict__ cont, const DecSection* __restrict__ sec,
                                                         int nsec, u64* __restrict__ syms, u32* __restrict__ scratch,
                                                         const int* __restrict__ ids, int* __restrict__ err) {
    extern __shared__ __align__(16) u8 dec_smem[];
    const int lane = threadIdx.x;
    const int si = ids ? ids[blockIdx.x] : static_cast<int>(blockIdx.x);
    if (si >= nsec) return;
    const DecSection d = sec[si];
    const u8* p = cont + d.ent_off;
    const u32 n = d.nsym;
    if (n == 0) return;
    u64* out = syms + d.sym_off;
    if (p[0] == 1) {  // semi-static rANS (entropy.cpp:290-421), lane 0
        if (lane != 0) return;
        const u8* in = p + 5;
        const u64 len = d.ent_len - 5;
        u64 pos = 0;
        auto varint = [&](u64& v) {
            v = 0;
            for (unsigned sh = 0;; sh += 7) {
                if (pos >= len || sh > 63) return false;
                const u8 b = in[pos++];
                v |= static_cast<u64>(b & 0x7F) << sh;
                if (!(b & 0x80)) return true;
            }
        };
        u64 ntab = 0, bits = 0;
        if (!varint(ntab) || !varint(bits) || bits > 20 || ntab == 0) return dec_fail(err, kDecErrEntropy);
        u64* tsym = reinterpret_cast<u64*>(scratch + d.scratch_off);  // ntab symbols
        u32* tf = reinterpret_cast<u32*>(tsym + ntab);                // ntab freqs
        u32* tc = tf + ntab;                                           // ntab + 1 cumulative
        u64 prev = 0, total = 0;
        tc[0] = 0;
        for (u64 i = 0; i < ntab; ++i) {
            u64 ds = 0, f = 0;
            if (!varint(ds) || !varint(f)) return dec_fail(err, kDecErrEntropy);
            prev += ds;
            tsym[i] = prev;
            tf[i] = static_cast<u32>(f);
            total += f;
            tc[i + 1] = static_cast<u32>(total);
        }
        if (total != (u64{1} << bits) || pos + 8 > len) return dec_fail(err, kDecErrEntropy);
        u64 x = 0;
        for (int i = 0; i < 8; ++i) x |= static_cast<u64>(in[pos + i]) << (8 * i);
        pos += 8;
        const u64 mask = (u64{1} << bits) - 1;
        for (u32 q = 0; q < n; ++q) {
            const u32 slot = static_cast<u32>(x & mask);
            u64 lo = 0, hi = ntab;  // largest j with tc[j] <= slot
            while (hi - lo > 1) {
                const u64 mid = (lo + hi) / 2;
                if (tc[mid] <= slot) lo = mid;
                else hi = mid;
            }
            out[q] = tsym[lo];
            x = static_cast<u64>(tf[lo]) * (x >> bits) + slot - tc[lo];
            while (x < (u64{1} << 31)) {
                if (pos + 4 > len) return dec_fail(err, kDecErrEntropy);
                const u32 w = dec_le32(in + pos);
                pos += 4;
                x = (x << 32) | w;
            }
        }
        return;
    }
    if (p[0] != 0) return dec_fail(err, kDecErrCoder);
    // adaptive range coder
    const u32 cap = kShared ? kDecCap : d.cap;
    u32* base = kShared ? reinterpret_cast<u32*>(dec_smem) : scratch + d.scratch_off;
    u32* cnt = base;
    u32* l1 = cnt + cap;
    u32* l2 = l1 + (cap / 32 + 1);
    u64* val = reinterpret_cast<u64*>(base + ((cap + (cap / 32 + 1) + (cap / 1024 + 1) + 1) & ~1u));
    for (u32 i = lane; i < cap; i += 32) cnt[i] = 0;
    for (u32 i = lane; i <= cap / 32; i += 32) l1[i] = 0;
    for (u32 i = lane; i <= cap / 1024; i += 32) l2[i] = 0;
    __syncwarp();
    if (lane == 0) {
        cnt[0] = 1;
        l1[0] = 1;
        l2[0] = 1;
        val[0] = 0;
    }
    __syncwarp();
    const u8* body = p + 5;
    const u64 blen = d.ent_len - 5;
    u64 pos = 0;
    auto next = [&]() -> u32 { return pos < blen ? body[pos++] : 0u; };
    u32 range = 0xFFFFFFFFu, code = 0;
    for (int i = 0; i < 5; ++i) code = (code << 8) | next();
    u32 nsym = 1, total = 1;
    auto norm = [&]() {
        while (range < (1u << 24)) {
            code = (code << 8) | next();
            range <<= 8;
        }
    };
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
            u32 bs = c;
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
    // first index in [0, m) whose inclusive prefix exceeds t; the prefix below it in *below
    auto find = [&](const u32* a, u32 m, u32 t, u32* below) -> u32 {
        u32 acc = 0;
        for (u32 b0 = 0; b0 < m; b0 += 32) {
            const u32 v = b0 + lane < m ? a[b0 + lane] : 0u;
            u32 inc = v;
            for (int o = 1; o < 32; o <<= 1) {
                const u32 y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, acc + inc > t);
            if (hit) {
                const int f = __ffs(hit) - 1;
                const u32 ex = __shfl_sync(0xffffffffu, inc - v, f);
                *below = acc + ex;
                return b0 + f;
            }
            acc += __shfl_sync(0xffffffffu, inc, 31);
        }
        *below = acc;
        return m;  // not found (corrupt stream)
    };
    for (u32 q = 0; q < n; ++q) {
        range /= total;
        u32 t = code / range;
        if (t >= total) t = total - 1;
        // locate: 1024-blocks, then 32-blocks, then entries
        u32 b2b = 0, b1b = 0, cb = 0;
        // a level with a single block holds the whole remaining range: no search
        const u32 n2 = (nsym + 1023) / 1024;
        const u32 b2 = n2 == 1 ? 0u : find(l2, n2, t, &b2b);
        const u32 lo1 = b2 * 32, n1 = min((nsym + 31) / 32 - lo1, 32u);
        const u32 b1 = b2 < n2 ? (n1 == 1 ? 0u : find(l1 + lo1, n1, t - b2b, &b1b)) : n1;
        const u32 lo0 = (lo1 + b1) * 32, n0 = min(nsym - lo0, 32u);
        const u32 c0 = b1 < n1 ? find(cnt + lo0, n0, t - b2b - b1b, &cb) : n0;
        if (b2 >= n2 || b1 >= n1 || c0 >= n0) return dec_fail(err, kDecErrEntropy);
        const u32 i = lo0 + c0;
        const u32 cum = b2b + b1b + cb, f = cnt[i];
        code -= cum * range;
        range *= f;
        norm();
        u64 sv;
        if (i == 0) {  // escape: 32 raw bits as decode(bit, 1, 2)
            // per bit: range >>= 1; bit = min(code / range, 1); code -= bit range; norm().
            // With range in [2^24, 2^32) exactly k = floor(log2 range) - 23 halvings
            // happen before the next normalisation, so up to k bits go at once, each
            // a compare instead of a divide (same arithmetic as the encoder's groups).
            u64 v = 0;
            int left = 32;
            while (left > 0) {
                const int k = min(left, (31 - __clz(static_cast<int>(range))) - 23);
#pragma unroll
                for (int j = 1; j <= 8; ++j)
                    if (j <= k) {
                        const u32 rj = range >> j;
                        const u32 bit = code >= rj ? 1u : 0u;
                        code -= bit ? rj : 0u;
                        v = (v << 1) | bit;
                    }
                range >>= k;
                left -= k;
                norm();
            }
            sv = v;
            if (total + 32 >= (1u << 16)) halve();
            if (nsym >= cap) return dec_fail(err, kDecErrModel);
            __syncwarp();
            if (lane == 0) {
                val[nsym] = sv;
                cnt[nsym] = 32;
                l1[nsym >> 5] += 32;
                l2[nsym >> 10] += 32;
            }
            ++nsym;
        } else {
            sv = val[i];
            if (total + 32 >= (1u << 16)) halve();
            __syncwarp();
            if (lane == 0) {
                cnt[i] += 32;
                l1[i >> 5] += 32;
                l2[i >> 10] += 32;
            }
        }
        total += 32;
        __syncwarp();
        if (lane == 0) out[q] = sv;
    }
}

// ---------------------------------------------------------------- plane / block reconstruction
constexpr int kDsT = 256;
constexpr int kDsI = 8;  // coefficients per thread in a plane pass

__device__ __forceinline__ u32 dec_cta_excl_scan(u32 v, u32* sh, u32& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u32 x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        u32 run = 0;
        for (int i = 0; i < kDsT / 32; ++i) {
            const u32 t = sh[i];
            sh[i] = run;
            run += t;
        }
        sh[kDsT / 32] = run;
    }
    __syncthreads();
    total = sh[kDsT / 32];
    return sh[w] + x - v;
}

__global__ void __launch_bounds__(kDsT) dec_stream_kernel(const u8* __restrict__ cont,
                                                         const DecStream* __restrict__ streams,
                                                         const DecBlock* __restrict__ blocks,
                                                         const DecSection* __restrict__ sec,
                                                         const u64* __restrict__ syms, u64* __restrict__ mag,
                                                         u8* __restrict__ neg, u8* __restrict__ pe,
                                                         u8* __restrict__ colbits, int* __restrict__ err) {
    __shared__ u32 shs[kDsT / 32 + 1];
    const DecBlock bk = blocks[blockIdx.x];
    const DecStream st = streams[bk.stream];
    const u64 lo = bk.lo, hi = bk.hi, bn = hi - lo;
    u64* m = mag + st.out_off;
    u8* ng = neg + st.out_off;
    u8* pl = pe + st.out_off;
    u8* col = colbits + st.out_off;  // per-block scratch: the leading column of the current plane
    for (u64 i = lo + threadIdx.x; i < hi; i += kDsT) {
        m[i] = 0;
        ng[i] = 0;
        pl[i] = 0;
    }
    __syncthreads();
    for (u32 rel = 0; rel < st.nplanes; ++rel) {
        const int p = 63 - static_cast<int>(rel);
        const bool last = p == st.last_plane;
        const u64 ls = last ? st.stops_lead[bk.b] : ~u64{0};
        const u64 ts = last ? st.stops_trail[bk.b] : ~u64{0};
        const DecSection d = sec[st.sec_off + static_cast<u64>(rel) * st.nb + bk.b];
        // still-insignificant coefficients of the block
        u32 ins = 0;
        for (u64 i = lo + threadIdx.x; i < hi; i += kDsT) ins += m[i] == 0;
        for (int o = 16; o > 0; o >>= 1) ins += __shfl_xor_sync(0xffffffffu, ins, o);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) shs[threadIdx.x >> 5] = ins;
        __syncthreads();
        u64 insig = 0;
        for (int w = 0; w < kDsT / 32; ++w) insig += shs[w];
        const u64 clen = insig < ls ? insig : ls;
        // leading column from the runs: ones at prefix(runs) + index
        if (clen > 0) {
            if (d.elen == 0) {
                if (threadIdx.x == 0) dec_fail(err, kDecErrMissingColumn);
                return;
            }
            for (u64 i = threadIdx.x; i < clen; i += kDsT) col[lo + i] = 0;
            __syncthreads();
            const u64* runs = syms + d.sym_off;
            const u32 R = d.nsym;
            if (R == 0) {
                if (threadIdx.x == 0) dec_fail(err, kDecErrRle);
                return;
            }
            u64 carry = 0;
            for (u32 r0 = 0; r0 < R; r0 += kDsT) {
                const u32 r = r0 + threadIdx.x;
                const u64 v = r < R ? runs[r] : 0;
                // inclusive scan of run lengths (u64) over the CTA
                u64 x = v;
                for (int o = 1; o < 32; o <<= 1) {
                    const u64 y = __shfl_up_sync(0xffffffffu, x, o);
                    if ((threadIdx.x & 31) >= o) x += y;
                }
                __shared__ u64 wsum[kDsT / 32 + 1];
                __syncthreads();
                if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
                __syncthreads();
                if (threadIdx.x == 0) {
                    u64 run = 0;
                    for (int i = 0; i < kDsT / 32; ++i) {
                        const u64 t = wsum[i];
                        wsum[i] = run;
                        run += t;
                    }
                    wsum[kDsT / 32] = run;
                }
                __syncthreads();
                const u64 incl = carry + wsum[threadIdx.x >> 5] + x;
                if (r + 1 < R) {  // a one follows every run except the last
                    const u64 pos = incl + r;
                    if (pos < clen) col[lo + pos] = 1;
                    else dec_fail(err, kDecErrRle);
                } else if (r + 1 == R && incl + r != clen) {
                    dec_fail(err, kDecErrRle);
                }
                carry += wsum[kDsT / 32];
                __syncthreads();
            }
            __syncthreads();
        }
        // coefficient pass: ranks among insignificant / significant / bit consumers.
        // Each thread owns kDsI consecutive coefficients of a kDsT*kDsI chunk, so a
        // chunk costs two CTA scans: (insignificant, significant) packed in one
        // u32, then the bit consumers
        const u8* raw = cont + d.raw_off;
        const u64 rawbits = static_cast<u64>(d.raw_len) * 8;
        u64 ins_base = 0, sig_base = 0, raw_base = 0;
        for (u64 c0 = lo; c0 < hi; c0 += static_cast<u64>(kDsT) * kDsI) {
            const u64 i0 = c0 + static_cast<u64>(threadIdx.x) * kDsI;
            u64 mv[kDsI];
            u32 nin = 0, nsg = 0;
#pragma unroll
            for (int j = 0; j < kDsI; ++j) {
                const bool in = i0 + j < hi;
                mv[j] = in ? m[i0 + j] : 0;
                nin += (in && mv[j] == 0) ? 1u : 0u;
                nsg += mv[j] != 0 ? 1u : 0u;
            }
            u32 tot_is = 0, tot_raw = 0;
            const u32 ex = dec_cta_excl_scan(nin | (nsg << 16), shs, tot_is);
            u64 lu = ins_base + (ex & 0xFFFFu), tu = sig_base + (ex >> 16);
            u32 cons = 0, refm = 0;  // per-item bit masks: consumes a raw bit / is a refinement
#pragma unroll
            for (int j = 0; j < kDsI; ++j) {
                if (i0 + j >= hi) continue;
                if (mv[j] != 0) {
                    if (tu < ts) {
                        cons |= 1u << j;
                        refm |= 1u << j;
                    }
                    ++tu;
                } else {
                    if (lu < ls && lu < clen && col[lo + lu] != 0) cons |= 1u << j;
                    ++lu;
                }
            }
            u64 bpos = raw_base + dec_cta_excl_scan(static_cast<u32>(__popc(cons)), shs, tot_raw);
#pragma unroll
            for (int j = 0; j < kDsI; ++j) {
                if (!(cons >> j & 1u)) continue;
                if (bpos >= rawbits) {
                    dec_fail(err, kDecErrBits);
                } else {
                    const bool bit = (raw[bpos >> 3] >> (7 - (bpos & 7))) & 1u;
                    if (refm >> j & 1u) {
                        if (bit) m[i0 + j] = mv[j] | (u64{1} << p);
                    } else {
                        m[i0 + j] = u64{1} << p;
                        ng[i0 + j] = bit ? 1 : 0;
                    }
                    pl[i0 + j] = static_cast<u8>(p);
                }
                ++bpos;
            }
            ins_base += tot_is & 0xFFFFu;
            sig_base += tot_is >> 16;
            raw_base += tot_raw;
            __syncthreads();
        }
        __syncthreads();
    }
    for (u64 i = lo + threadIdx.x; i < hi; i += kDsT)
        if (m[i] != 0 && pl[i] >= 1) m[i] += u64{1} << (pl[i] - 1);
    (void)bn;
}

// core value = +-ldexp(mag, -k)
__global__ void dequant_kernel(const u64* __restrict__ mag, const u8* __restrict__ neg, u64 n, int k,
                               double* __restrict__ out, const u64* __restrict__ order) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double v = scalbn(__ull2double_rn(mag[i]), -k);
        out[order ? order[i] : i] = neg[i] ? -v : v;
    }
}

template <class N>
__global__ void emit_kernel(const double* __restrict__ x, u64 n, N* __restrict__ out) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double v = x[i];
        if constexpr (std::is_integral_v<N>) {
            const double lo = static_cast<double>(std::numeric_limits<N>::min());
            const double hi = static_cast<double>(std::numeric_limits<N>::max());
            const double r = nearbyint(v);
            N o;
            if (r <= lo) o = std::numeric_limits<N>::min();
            else if (r >= hi) o = std::numeric_limits<N>::max();
            else o = static_cast<N>(r);
            out[i] = o;
        } else {
            out[i] = static_cast<N>(v);
        }
    }
}

}  // namespace

void decode_entropy(const u8* cont, const DecSection* sec_dev, const std::vector<DecSection>& sec, u64* syms,
                    u32* scratch, int* err, cudaStream_t s) {
    const int ns = static_cast<int>(sec.size());
    if (ns == 0) return;
    std::vector<int> small_ids, big_ids;
    for (int i = 0; i < ns; ++i) {
        if (sec[i].nsym == 0) continue;
        if (sec[i].cap <= kDecCap) small_ids.push_back(i);
        else big_ids.push_back(i);
    }
    TCB_ONCE_PER_DEVICE(cudaFuncSetAttribute(dec_entropy_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(dec_model_words(kDecCap) * 4 + 16)));
    for (int pass = 0; pass < 2; ++pass) {
        const auto& ids = pass == 0 ? small_ids : big_ids;
        if (ids.empty()) continue;
        DevBuf<int> did(ids.size(), s);
        did.upload(ids.data(), ids.size());
        if (pass == 0)
            dec_entropy_kernel<true><<<static_cast<unsigned>(ids.size()), 32, dec_model_words(kDecCap) * 4 + 16, s>>>(
                cont, sec_dev, ns, syms, scratch, did.p, err);
        else
            dec_entropy_kernel<false><<<static_cast<unsigned>(ids.size()), 32, 0, s>>>(cont, sec_dev, ns, syms,
                                                                                      scratch, did.p, err);
        count_launch();
        TCB_LAUNCH();
    }
}

u64 decode_model_words(u32 cap) { return dec_model_words(cap); }

void decode_streams(const u8* cont, const DecStream* streams, const DecBlock* blocks, u64 nblocks,
                    const DecSection* sec, const u64* syms, u64* mag, u8* neg, u8* pe, u8* colbits, int* err,
                    cudaStream_t s) {
    if (nblocks == 0) return;
    dec_stream_kernel<<<static_cast<unsigned>(nblocks), kDsT, 0, s>>>(cont, streams, blocks, sec, syms, mag, neg, pe,
                                                                     colbits, err);
    count_launch();
    TCB_LAUNCH();
}

void dequantize(const u64* mag, const u8* neg, u64 n, int k, double* out, cudaStream_t s, const u64* order) {
    if (n == 0) return;
    dequant_kernel<<<std::min<unsigned>(cdiv(n, 256), 4 * sm_count()), 256, 0, s>>>(mag, neg, n, k, out, order);
    count_launch();
    TCB_LAUNCH();
}

void emit_dtype(const double* x, u64 n, int dtype, void* out, cudaStream_t s) {
    if (n == 0) return;
    const unsigned g = std::min<unsigned>(cdiv(n, 256), 4 * sm_count());
    switch (dtype) {
        case 0: emit_kernel<int8_t><<<g, 256, 0, s>>>(x, n, static_cast<int8_t*>(out)); break;
        case 1: emit_kernel<uint8_t><<<g, 256, 0, s>>>(x, n, static_cast<uint8_t*>(out)); break;
        case 2: emit_kernel<int16_t><<<g, 256, 0, s>>>(x, n, static_cast<int16_t*>(out)); break;
        case 3: emit_kernel<uint16_t><<<g, 256, 0, s>>>(x, n, static_cast<uint16_t*>(out)); break;
        case 4: emit_kernel<int32_t><<<g, 256, 0, s>>>(x, n, static_cast<int32_t*>(out)); break;
        case 5: emit_kernel<uint32_t><<<g, 256, 0, s>>>(x, n, static_cast<uint32_t*>(out)); break;
        case 6: emit_kernel<int64_t><<<g, 256, 0, s>>>(x, n, static_cast<int64_t*>(out)); break;
        case 7: emit_kernel<uint64_t><<<g, 256, 0, s>>>(x, n, static_cast<uint64_t*>(out)); break;
        case 8: emit_kernel<float><<<g, 256, 0, s>>>(x, n, static_cast<float*>(out)); break;
        case 9: emit_kernel<double><<<g, 256, 0, s>>>(x, n, static_cast<double*>(out)); break;
        default: throw Error("emit: unknown dtype");
    }
    count_launch();
    TCB_LAUNCH();
}

}  // namespace tcb
