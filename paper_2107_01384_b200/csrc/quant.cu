// Core quantisation (core_codec.cpp:55-93), dead slices (:510-523) and the
// Householder sign fold (pipeline.cpp:161-175).  Integer-exact kernels.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

#include "kernels.cuh"
#include "quant.cuh"

namespace tcb {

namespace {

// m = nearbyint(ldexp(|x|, k)) (round-half-even), sign = x < 0
__global__ void quantize_kernel(const double* __restrict__ x, u64 n, int k, u64* __restrict__ mag,
                                u8* __restrict__ neg, const u64* __restrict__ order) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double v = x[order ? order[i] : i];
        mag[i] = __double2ull_rn(scalbn(fabs(v), k));
        neg[i] = v < 0.0 ? 1 : 0;
    }
}

// Serial replay of the per-slice accumulation in vectorisation (lex) order:
// one thread per (axis, index); slice elements are visited in increasing flat
// position, each term (double)m*(double)m added with round-to-nearest.
__global__ void slice_norm_kernel(const u64* __restrict__ mag, const u64* __restrict__ shape, int d, u64 total,
                                  double down, double* __restrict__ out) {
    const u64 t = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= total) return;
    int a = 0;
    u64 base = 0;
    while (t >= base + shape[a]) {
        base += shape[a];
        ++a;
    }
    const u64 idx = t - base;
    u64 inner = 1, outer = 1;
    for (int i = a + 1; i < d; ++i) inner *= shape[i];
    for (int i = 0; i < a; ++i) outer *= shape[i];
    const u64 ext = shape[a];
    // the reference's serial order (outer, then inner), 8 elements per step: their
    // loads are issued together so the dependent adds do not wait on memory
    double s = 0.0;
    const u64 cnt = outer * inner;
    u64 o = 0, q = 0;  // position of element j in (outer, inner)
    for (u64 j0 = 0; j0 < cnt; j0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            v[u] = j0 + u < cnt ? __ull2double_rn(mag[(o * ext + idx) * inner + q]) : 0.0;
            if (++q == inner) {
                q = 0;
                ++o;
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (j0 + u < cnt) s = __dadd_rn(s, __dmul_rn(v[u], v[u]));
    }
    out[t] = __dsqrt_rn(__dmul_rn(s, down));
}

// The same serial slice sums, one CTA per slice, for large slices: the CTA
// stages the next chunk of squares in shared memory (the divisions and the
// strided loads spread over the CTA) while thread 0 runs the dependent add
// chain over the current chunk.
constexpr int kSnThreads = 256, kSnChunk = 2048;
__global__ void __launch_bounds__(kSnThreads) slice_norm_cta_kernel(const u64* __restrict__ mag,
                                                                    const u64* __restrict__ shape, int d,
                                                                    double down, double* __restrict__ out) {
    __shared__ double buf[2][kSnChunk];
    const u64 t = blockIdx.x;
    int a = 0;
    u64 base = 0;
    while (t >= base + shape[a]) {
        base += shape[a];
        ++a;
    }
    const u64 idx = t - base;
    u64 inner = 1, outer = 1;
    for (int i = a + 1; i < d; ++i) inner *= shape[i];
    for (int i = 0; i < a; ++i) outer *= shape[i];
    const u64 ext = shape[a], cnt = outer * inner, nchunk = (cnt + kSnChunk - 1) / kSnChunk;
    auto fill = [&](u64 c, int b) {
        for (int q = threadIdx.x; q < kSnChunk; q += blockDim.x) {
            const u64 j = c * kSnChunk + q;
            double sq = 0.0;
            if (j < cnt) {
                const u64 o = j / inner, r = j - o * inner;
                const double v = __ull2double_rn(mag[(o * ext + idx) * inner + r]);
                sq = __dmul_rn(v, v);
            }
            buf[b][q] = sq;
        }
    };
    double s = 0.0;
    if (nchunk) fill(0, 0);
    __syncthreads();
    for (u64 c = 0; c < nchunk; ++c) {
        const int b = static_cast<int>(c & 1);
        if (c + 1 < nchunk) fill(c + 1, b ^ 1);
        if (threadIdx.x == 0) {
            const u64 rem = cnt - c * kSnChunk;
            const int m = static_cast<int>(rem < kSnChunk ? rem : kSnChunk);
            for (int q0 = 0; q0 < m; q0 += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = buf[b][q0 + u];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (q0 + u < m) s = __dadd_rn(s, v[u]);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[t] = __dsqrt_rn(__dmul_rn(s, down));
}

// I = u32 when the core has fewer than 2^32 coefficients (32-bit index division)
template <class I>
__global__ void dead_kernel(const u64* __restrict__ dec, u64 n, const u64* __restrict__ meta /* shape, stride, off */,
                            int d, u8* __restrict__ dead, const u64* __restrict__ order) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 v = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
        if (dec[v] == 0) continue;
        const I pos = static_cast<I>(order ? order[v] : v);
        for (int a = 0; a < d; ++a) {
            const I idx = (pos / static_cast<I>(meta[d + a])) % static_cast<I>(meta[a]);
            u8* q = dead + meta[2 * d + a] + idx;
            if (*q) *q = 0;  // most slices are live: read before write
        }
    }
}

template <class I>
__global__ void signfold_kernel(u8* __restrict__ neg, u64 n, const u64* __restrict__ meta, int d,
                                const signed char* __restrict__ flips /* concatenated per storage axis */,
                                const u64* __restrict__ order) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 v = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
        const I pos = static_cast<I>(order ? order[v] : v);
        u8 par = 0;
        for (int a = 0; a < d; ++a) {
            const I idx = (pos / static_cast<I>(meta[d + a])) % static_cast<I>(meta[a]);
            par ^= flips[meta[2 * d + a] + idx] < 0 ? 1 : 0;
        }
        neg[v] ^= par;
    }
}

// Lexicographic order (no order map): a CTA per run of rows along the last
// axis -- the other axes' slice indices (and their flips) are the row's, found
// once per row, and the last axis is a coalesced byte pass.
__global__ void signfold_rows_kernel(u8* __restrict__ neg, u64 nrows, const u64* __restrict__ meta, int d,
                                     const signed char* __restrict__ flips) {
    const u64 last = meta[d - 1];
    const signed char* fl = flips + meta[3 * d - 1];
    for (u64 row = blockIdx.x; row < nrows; row += gridDim.x) {
        u8 par = 0;
        u64 rem = row;
        for (int a = d - 2; a >= 0; --a) {
            const u64 e = meta[a];
            u64 q, r;
            if (rem < (u64{1} << 32) && e < (u64{1} << 32)) {  // 32-bit division where it fits
                q = static_cast<u32>(rem) / static_cast<u32>(e);
                r = static_cast<u32>(rem) - static_cast<u32>(q) * static_cast<u32>(e);
            } else {
                q = rem / e;
                r = rem - q * e;
            }
            par ^= flips[meta[2 * d + a] + r] < 0 ? 1 : 0;
            rem = q;
        }
        u8* q8 = neg + row * last;
        for (u64 k = threadIdx.x; k < last; k += blockDim.x) q8[k] ^= par ^ (fl[k] < 0 ? 1 : 0);
    }
}

// 8 rows per step: one barrier per step decides which rows are live
__global__ void dead_rows_kernel(const u64* __restrict__ dec, u64 nrows, const u64* __restrict__ meta, int d,
                                 u8* __restrict__ dead) {
    __shared__ int live[8];
    const u64 last = meta[d - 1];
    u8* dl = dead + meta[3 * d - 1];
    for (u64 row0 = static_cast<u64>(blockIdx.x) * 8; row0 < nrows; row0 += static_cast<u64>(gridDim.x) * 8) {
        if (threadIdx.x < 8) live[threadIdx.x] = 0;
        __syncthreads();
        const u64 nr = min(u64{8}, nrows - row0);
        for (u64 rr = 0; rr < nr; ++rr) {
            const u64* q = dec + (row0 + rr) * last;
            bool any = false;
            for (u64 k = threadIdx.x; k < last; k += blockDim.x)
                if (q[k]) {
                    any = true;
                    if (dl[k]) dl[k] = 0;  // most slices are live: read before write
                }
            if (any) live[rr] = 1;
        }
        __syncthreads();
        if (threadIdx.x < nr && live[threadIdx.x]) {
            u64 rem = row0 + threadIdx.x;
            for (int a = d - 2; a >= 0; --a) {
                u8* z = dead + meta[2 * d + a] + rem % meta[a];
                if (*z) *z = 0;
                rem /= meta[a];
            }
        }
        __syncthreads();
    }
}

// vectorize::OrderMap keys (vectorize.cpp:40-135): zigzag = (coordinate sum,
// row-major index), i.e. each anti-diagonal layer in lexicographic order;
// zorder = the Morton key (axis 0 most significant in each bit level).  A
// stable sort of the positions by key gives the iteration order.
__global__ void order_keys_kernel(const u64* __restrict__ meta, int d, u64 n, int method, unsigned levels,
                                  u64* __restrict__ keys, u64* __restrict__ pos) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 f = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; f < n; f += stride) {
        u64 key = 0;
        if (method == 1) {
            u64 sum = 0;
            for (int a = 0; a < d; ++a) sum += (f / meta[d + a]) % meta[a];
            key = sum * n + f;
        } else {
            for (int a = 0; a < d; ++a) {
                const u64 c = (f / meta[d + a]) % meta[a];
                for (unsigned t = 0; t < levels; ++t)
                    key |= ((c >> t) & 1u) << (t * static_cast<unsigned>(d) + static_cast<unsigned>(d - 1 - a));
            }
        }
        keys[f] = key;
        pos[f] = f;
    }
}

// coordinate along `axis` of each vectorised coefficient (sort key of its slice list)
__global__ void slice_keys_kernel(const u64* __restrict__ order, u64 n, u64 stride_a, u64 ext_a,
                                  u32* __restrict__ keys, u64* __restrict__ vals) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 v = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
        keys[v] = static_cast<u32>((order[v] / stride_a) % ext_a);
        vals[v] = v;
    }
}

// serial replay per slice over its coefficients in vectorised order (list
// segment [idx * per, (idx + 1) * per)), one thread per slice
__global__ void slice_norm_list_kernel(const u64* __restrict__ mag, const u64* __restrict__ list, u64 ext, u64 per,
                                       double down, double* __restrict__ out) {
    const u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= ext) return;
    double s = 0.0;
    const u64 j1 = (idx + 1) * per;
    for (u64 j0 = idx * per; j0 < j1; j0 += 8) {  // 8 gathers in flight per step
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = j0 + u < j1 ? __ull2double_rn(mag[list[j0 + u]]) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (j0 + u < j1) s = __dadd_rn(s, __dmul_rn(v[u], v[u]));
    }
    out[idx] = __dsqrt_rn(__dmul_rn(s, down));
}

template <class K>
void radix_sort_pairs(const K* kin, K* kout, const u64* vin, u64* vout, u64 n, int bits, cudaStream_t s) {
    size_t tmp = 0;
    TCB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, static_cast<int>(n), 0, bits, s));
    DevBuf<u8> t(std::max<size_t>(tmp, 1), s);
    TCB_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, kin, kout, vin, vout, static_cast<int>(n), 0, bits, s));
}

std::vector<u64> axis_meta(const std::vector<u64>& shape) {
    const int d = static_cast<int>(shape.size());
    std::vector<u64> meta(3 * d);
    u64 acc = 1;
    for (int i = d - 1; i >= 0; --i) {
        meta[d + i] = acc;
        acc *= shape[i];
    }
    u64 off = 0;
    for (int i = 0; i < d; ++i) {
        meta[i] = shape[i];
        meta[2 * d + i] = off;
        off += shape[i];
    }
    return meta;
}

}  // namespace

DevBuf<u64> order_map_device(int method, const std::vector<u64>& shape, cudaStream_t s) {
    if (method == 0) return DevBuf<u64>();
    if (method != 1 && method != 2) throw Error("vectorize: unknown method");
    const int d = static_cast<int>(shape.size());
    if (d == 0) throw Error("vectorize: empty shape");
    u64 n = 1;
    for (auto v : shape) n *= v;
    unsigned levels = 0;
    for (auto v : shape) {
        unsigned b = 0;
        while ((u64{1} << b) < v) ++b;
        levels = std::max(levels, b);
    }
    if (method == 2 && static_cast<u64>(levels) * d > 63)
        throw Error("vectorize: shape too large for 64-bit Morton keys");
    if (n > 0x7FFFFFFFull) throw Error("vectorize: core too large for the device order map");
    const auto meta = axis_meta(shape);
    DevBuf<u64> dm(meta.size(), s);
    dm.upload(meta.data(), meta.size());
    DevBuf<u64> keys(n, s), keys2(n, s), pos(n, s), order(n, s);
    order_keys_kernel<<<std::min<unsigned>(cdiv(n, 256), 4 * sm_count()), 256, 0, s>>>(dm.p, d, n, method, levels,
                                                                                       keys.p, pos.p);
    count_launch();
    TCB_LAUNCH();
    radix_sort_pairs<u64>(keys.p, keys2.p, pos.p, order.p, n, 64, s);
    return order;
}

void quantize_f64(const double* x, u64 n, int k, u64* mag, u8* neg, cudaStream_t s, const u64* order) {
    ProfScope prof_scope(kQuant, s);
    if (n == 0) return;
    quantize_kernel<<<grid_for(n, 256, 4, 8), 256, 0, s>>>(x, n, k, mag, neg, order);
    count_launch();
    TCB_LAUNCH();
}

void slice_norms(const u64* mag, const std::vector<u64>& shape, double down, double* out, cudaStream_t s,
                 const u64* order) {
    ProfScope prof_scope(kQuant, s);
    u64 total = 0, n = 1;
    for (auto v : shape) {
        total += v;
        n *= v;
    }
    if (!order) {
        DevBuf<u64> sh(shape.size(), s);
        sh.upload(shape.data(), shape.size());
        if (n / std::max<u64>(1, *std::min_element(shape.begin(), shape.end())) >= 16384) {  // large slices
            slice_norm_cta_kernel<<<static_cast<unsigned>(total), kSnThreads, 0, s>>>(
                mag, sh.p, static_cast<int>(shape.size()), down, out);
            count_launch();
            TCB_LAUNCH();
            return;
        }
        slice_norm_kernel<<<cdiv(total, 64), 64, 0, s>>>(mag, sh.p, static_cast<int>(shape.size()), total, down,
                                                         out);
        count_launch();
        TCB_LAUNCH();
        return;
    }
    // non-lexicographic: each slice's coefficients in vectorised order (stable sort by coordinate)
    const auto meta = axis_meta(shape);
    const int d = static_cast<int>(shape.size());
    DevBuf<u32> k1(n, s), k2(n, s);
    DevBuf<u64> v1(n, s), list(n, s);
    u64 off = 0;
    for (int a = 0; a < d; ++a) {
        slice_keys_kernel<<<std::min<unsigned>(cdiv(n, 256), 4 * sm_count()), 256, 0, s>>>(order, n, meta[d + a],
                                                                                           shape[a], k1.p, v1.p);
        int bits = 1;
        while ((u64{1} << bits) < shape[a]) ++bits;
        radix_sort_pairs<u32>(k1.p, k2.p, v1.p, list.p, n, bits, s);
        slice_norm_list_kernel<<<cdiv(shape[a], 64), 64, 0, s>>>(mag, list.p, shape[a], n / shape[a], down,
                                                                 out + off);
        count_launch(2);
        TCB_LAUNCH();
        off += shape[a];
    }
}

std::vector<u8> dead_slices(const u64* dec, const std::vector<u64>& shape, cudaStream_t s, const u64* order) {
    ProfScope prof_scope(kQuant, s);
    const auto meta = axis_meta(shape);
    u64 n = 1, total = 0;
    for (auto v : shape) {
        n *= v;
        total += v;
    }
    DevBuf<u64> dm(meta.size(), s);
    dm.upload(meta.data(), meta.size());
    DevBuf<u8> dead(total, s);
    TCB_CUDA(cudaMemsetAsync(dead.p, 1, total, s));
    if (!order && !shape.empty() && n > 0) {
        const u64 nrows = n / shape.back();
        dead_rows_kernel<<<static_cast<unsigned>(std::min<u64>(cdiv(nrows, 8), 148 * 16)), 256, 0, s>>>(
            dec, nrows, dm.p, static_cast<int>(shape.size()), dead.p);
    } else if (n < (u64{1} << 32))
        dead_kernel<u32><<<grid_for(n, 256, 4, 4), 256, 0, s>>>(dec, n, dm.p, static_cast<int>(shape.size()), dead.p,
                                                                 order);
    else
        dead_kernel<u64><<<grid_for(n, 256, 4, 4), 256, 0, s>>>(dec, n, dm.p, static_cast<int>(shape.size()), dead.p,
                                                                 order);
    count_launch();
    TCB_LAUNCH();
    return dead.to_host();
}

void sign_fold(u8* neg, const std::vector<u64>& shape, const std::vector<signed char>& flips_by_axis,
               cudaStream_t s, const u64* order) {
    ProfScope prof_scope(kQuant, s);
    const auto meta = axis_meta(shape);
    u64 n = 1;
    for (auto v : shape) n *= v;
    DevBuf<u64> dm(meta.size(), s);
    dm.upload(meta.data(), meta.size());
    DevBuf<signed char> fl(flips_by_axis.size(), s);
    fl.upload(flips_by_axis.data(), flips_by_axis.size());
    if (!order && !shape.empty() && n > 0) {
        const u64 nrows = n / shape.back();
        signfold_rows_kernel<<<static_cast<unsigned>(std::min<u64>(nrows, 148 * 16)), 128, 0, s>>>(
            neg, nrows, dm.p, static_cast<int>(shape.size()), fl.p);
    } else if (n < (u64{1} << 32))
        signfold_kernel<u32><<<grid_for(n, 256, 4, 4), 256, 0, s>>>(neg, n, dm.p, static_cast<int>(shape.size()), fl.p,
                                                                     order);
    else
        signfold_kernel<u64><<<grid_for(n, 256, 4, 4), 256, 0, s>>>(neg, n, dm.p, static_cast<int>(shape.size()), fl.p,
                                                                     order);
    count_launch();
    TCB_LAUNCH();
}

}  // namespace tcb
