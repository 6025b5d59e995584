// Ingest: source dtype -> T cast (container.cpp:51-94), finite check
// (kernels_avx2.cpp:68-95), ||A||^2 (tensor.cpp:152-155), exact max |x|, and
// the single row-major axis permutation (tensor.cpp:105-144).
// All HBM-bound: 16-byte vector loads, grid = k x 148 SMs, fixed reduction tree.
#include <cmath>
#include <cstdint>

#include <cstring>

#include "kernels.cuh"

namespace tcb {

namespace {

template <class S>
__device__ __forceinline__ double as_d(S v) { return static_cast<double>(v); }

template <class S, class T>
__global__ void cast_kernel(const S* __restrict__ src, T* __restrict__ dst, u64 n) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = static_cast<T>(src[i]);
}

// double -> double fast path: 16-byte copies
__global__ void copy16_kernel(const double2* __restrict__ src, double2* __restrict__ dst, u64 n2) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n2; i += stride) dst[i] = src[i];
}

template <class T>
void cast_any(const void* src, int dtype, u64 n, T* dst, cudaStream_t s) {
    ProfScope prof_scope(kIngest, s);
    const unsigned grid = static_cast<unsigned>(grid_for(n, 256, 4, 8)), blk = 256;
    switch (dtype) {
        case 0: cast_kernel<<<grid, blk, 0, s>>>(static_cast<const int8_t*>(src), dst, n); break;
        case 1: cast_kernel<<<grid, blk, 0, s>>>(static_cast<const uint8_t*>(src), dst, n); break;
        case 2: cast_kernel<<<grid, blk, 0, s>>>(static_cast<const int16_t*>(src), dst, n); break;
        case 3: cast_kernel<<<grid, blk, 0, s>>>(static_cast<const uint16_t*>(src), dst, n); break;
        case 4: cast_kernel<<<grid, blk, 0, s>>>(static_cast<const int32_t*>(src), dst, n); break;
        case 5: cast_kernel<<<grid, blk, 0, s>>>(static_cast<const uint32_t*>(src), dst, n); break;
        case 6: cast_kernel<<<grid, blk, 0, s>>>(static_cast<const int64_t*>(src), dst, n); break;
        case 7: cast_kernel<<<grid, blk, 0, s>>>(static_cast<const uint64_t*>(src), dst, n); break;
        case 8: cast_kernel<<<grid, blk, 0, s>>>(static_cast<const float*>(src), dst, n); break;
        case 9:
            if constexpr (std::is_same_v<T, double>) {
                if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 &&
                    n % 2 == 0) {
                    copy16_kernel<<<grid, blk, 0, s>>>(static_cast<const double2*>(src),
                                                       reinterpret_cast<double2*>(dst), n / 2);
                    break;
                }
            }
            cast_kernel<<<grid, blk, 0, s>>>(static_cast<const double*>(src), dst, n);
            break;
        default: throw Error("container: unknown dtype");
    }
    count_launch();
    TCB_LAUNCH();
}

constexpr int kRedThreads = 256;

// stage 1: per-CTA partial sums of squares + non-finite flag (fixed tree)
template <class T>
struct Vec16;  // 16-byte vector of T
template <>
struct Vec16<double> {
    using type = double2;
    static constexpr int W = 2;
    __device__ static void get(const double2& v, double (&o)[4]) { o[0] = v.x, o[1] = v.y, o[2] = o[3] = 0.0; }
};
template <>
struct Vec16<float> {
    using type = float4;
    static constexpr int W = 4;
    __device__ static void get(const float4& v, double (&o)[4]) { o[0] = v.x, o[1] = v.y, o[2] = v.z, o[3] = v.w; }
};

// sum of squares + non-finite flag; kVec: x is 16-byte aligned, so the body
// streams 16-byte vectors, four in flight per thread into four accumulators
template <class T, bool kVec>
__global__ void sumsq_stage1(const T* __restrict__ x, u64 n, double* __restrict__ part, int* __restrict__ bad) {
    __shared__ double sh[kRedThreads / 32];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int nonfinite = 0;
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    const u64 tid = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    u64 done = 0;
    if (kVec) {
        using V = typename Vec16<T>::type;
        constexpr int W = Vec16<T>::W;
        const V* xv = reinterpret_cast<const V*>(x);
        const u64 nv = n / W;
        u64 i = tid;
        for (; i + 3 * stride < nv; i += 4 * stride) {
            V v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldcs(xv + i + u * stride);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                double e[4];
                Vec16<T>::get(v[u], e);
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    nonfinite |= !isfinite(e[w]);
                    acc[u] = fma(e[w], e[w], acc[u]);
                }
            }
        }
        for (; i < nv; i += stride) {
            double e[4];
            Vec16<T>::get(__ldcs(xv + i), e);
#pragma unroll
            for (int w = 0; w < W; ++w) {
                nonfinite |= !isfinite(e[w]);
                acc[0] = fma(e[w], e[w], acc[0]);
            }
        }
        done = nv * W;
    }
    for (u64 i = done + tid; i < n; i += stride) {
        const double v = static_cast<double>(x[i]);
        nonfinite |= !isfinite(v);
        acc[1] = fma(v, v, acc[1]);
    }
    double t0 = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    for (int o = 16; o > 0; o >>= 1) t0 += __shfl_down_sync(0xffffffffu, t0, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t0;
    if (__syncthreads_or(nonfinite) && threadIdx.x == 0) *bad = 1;
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kRedThreads / 32; ++w) t += sh[w];
        part[blockIdx.x] = t;
    }
}

__global__ void sum_stage2(const double* __restrict__ part, int n, double* __restrict__ out) {
    __shared__ double sh[kRedThreads];
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) t += part[i];
    sh[threadIdx.x] = t;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

template <class T>
double sumsq_impl(const T* x, u64 n, bool* finite, cudaStream_t s) {
    ProfScope prof_scope(kIngest, s);
    const int grid = grid_for(n, kRedThreads, 8, 4);
    DevBuf<double> part(grid + 1, s);
    DevBuf<int> bad(1, s);
    bad.zero();
    if (reinterpret_cast<uintptr_t>(x) % 16 == 0)
        sumsq_stage1<T, true><<<grid, kRedThreads, 0, s>>>(x, n, part.p, bad.p);
    else
        sumsq_stage1<T, false><<<grid, kRedThreads, 0, s>>>(x, n, part.p, bad.p);
    sum_stage2<<<1, kRedThreads, 0, s>>>(part.p, grid, part.p + grid);
    count_launch(2);
    TCB_LAUNCH();
    double r = 0;
    int b = 0;
    d2h(&r, part.p + grid, sizeof(double), s);
    d2h(&b, bad.p, sizeof(int), s);
    stream_sync(s);
    if (finite) *finite = b == 0;
    return r;
}

__global__ void maxabs_stage1(const double* __restrict__ x, u64 n, double* __restrict__ part) {
    __shared__ double sh[kRedThreads / 32];
    double m = 0.0;
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        m = fmax(m, fabs(x[i]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kRedThreads / 32; ++w) t = fmax(t, sh[w]);
        part[blockIdx.x] = t;
    }
}

__global__ void max_stage2(const double* __restrict__ part, int n, double* __restrict__ out) {
    double m = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, part[i]);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t = fmax(t, sh[w]);
        *out = t;
    }
}

// gather permutation: output written contiguously (coalesced), input gathered
template <class T, int D>
__global__ void permute_kernel(const T* __restrict__ src, T* __restrict__ dst, u64 n,
                               const u64* __restrict__ meta /* out_shape[D], gather_stride[D] */) {
    u64 oshape[D], g[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        oshape[i] = meta[i];
        g[i] = meta[D + i];
    }
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 o = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; o < n; o += stride) {
        u64 rem = o, off = 0;
#pragma unroll
        for (int i = D - 1; i >= 0; --i) {
            const u64 idx = rem % oshape[i];
            rem /= oshape[i];
            off += idx * g[i];
        }
        dst[o] = src[off];
    }
}

// 3-D permutations that move the last axis: 32x32 smem tiles over the pair
// (input-last axis, output-last axis) so both sides stay coalesced.
template <class T>
__global__ void permute3_tiled(const T* __restrict__ src, T* __restrict__ dst, u64 s0, u64 s1, u64 s2,
                               int p0, int p1, int p2) {
    // output shape (S[p0], S[p1], S[p2]); input row-major (s0, s1, s2)
    __shared__ T tile[32][33];
    const u64 S[3] = {s0, s1, s2};
    const u64 in_st[3] = {s1 * s2, s2, 1};
    const int P[3] = {p0, p1, p2};
    // axis roles: a = input-last (2), b = output-last (P[2]); c = the remaining axis
    const int ax_b = P[2];
    const int ax_c = 3 - 2 - ax_b;  // since ax_b != 2 here
    const u64 nb = S[ax_b], na = S[2], nc = S[ax_c];
    const u64 tiles_a = (na + 31) / 32, tiles_b = (nb + 31) / 32;
    u64 t = blockIdx.x;
    const u64 ta = t % tiles_a;
    t /= tiles_a;
    const u64 tb = t % tiles_b;
    const u64 ic = t / tiles_b;
    if (ic >= nc) return;
    // output strides
    u64 out_st[3];
    out_st[2] = 1;
    out_st[1] = S[P[2]];
    out_st[0] = S[P[2]] * S[P[1]];
    u64 ost_of_axis[3];
    for (int i = 0; i < 3; ++i) ost_of_axis[P[i]] = out_st[i];
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const u64 ib = tb * 32 + j, ia = ta * 32 + threadIdx.x;
        if (ib < nb && ia < na) {
            const u64 off = ib * in_st[ax_b] + ia * in_st[2] + ic * in_st[ax_c];
            tile[j][threadIdx.x] = src[off];
        }
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const u64 ia = ta * 32 + j, ib = tb * 32 + threadIdx.x;
        if (ib < nb && ia < na) {
            const u64 off = ib * ost_of_axis[ax_b] + ia * ost_of_axis[2] + ic * ost_of_axis[ax_c];
            dst[off] = tile[threadIdx.x][j];
        }
    }
}

__global__ void precision_kernel(const void* __restrict__ src, int is_signed, u64 n, int* __restrict__ flag) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    int bad = 0;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        u64 mag;
        if (is_signed) {
            const long long v = static_cast<const long long*>(src)[i];
            mag = static_cast<u64>(v < 0 ? -(v + 1) : v);
        } else {
            mag = static_cast<const u64*>(src)[i];
        }
        bad |= mag > (u64{1} << 53);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

}  // namespace

bool ingest_precision_loss(const void* src, int dtype, u64 n, cudaStream_t s) {
    ProfScope prof_scope(kIngest, s);
    DevBuf<int> f(1, s);
    f.zero();
    precision_kernel<<<grid_for(n, 256, 4, 4), 256, 0, s>>>(src, dtype == 6 ? 1 : 0, n, f.p);
    count_launch();
    TCB_LAUNCH();
    return f.to_host()[0] != 0;
}

void ingest_cast(const void* src, int dtype, u64 n, double* dst, cudaStream_t s) { cast_any(src, dtype, n, dst, s); }
void ingest_cast_f32(const void* src, int dtype, u64 n, float* dst, cudaStream_t s) { cast_any(src, dtype, n, dst, s); }

double sum_squares(const double* x, u64 n, bool* finite, cudaStream_t s) { return sumsq_impl(x, n, finite, s); }
double sum_squares(const float* x, u64 n, bool* finite, cudaStream_t s) { return sumsq_impl(x, n, finite, s); }

// sse_between (tensor.cpp:147-164) of the ingested source and a reconstruction;
// with f32 both sides are rounded to float first (the reference's float tensors).
template <bool kF32>
__global__ void sse_stage1(const double* __restrict__ a, const double* __restrict__ b, u64 n,
                           double* __restrict__ part) {
    __shared__ double sh[kRedThreads / 32];
    double acc = 0.0;
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        double x = __ldcs(a + i), y = __ldcs(b + i);
        if (kF32) {
            x = static_cast<double>(static_cast<float>(x));
            y = static_cast<double>(static_cast<float>(y));
        }
        const double e = x - y;
        acc = fma(e, e, acc);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kRedThreads / 32; ++w) t += sh[w];
        part[blockIdx.x] = t;
    }
}

double sse_between(const double* a, const double* b, u64 n, bool f32, cudaStream_t s) {
    const int grid = grid_for(n, kRedThreads, 4, 4);
    DevBuf<double> part(grid + 1, s);
    if (f32)
        sse_stage1<true><<<grid, kRedThreads, 0, s>>>(a, b, n, part.p);
    else
        sse_stage1<false><<<grid, kRedThreads, 0, s>>>(a, b, n, part.p);
    sum_stage2<<<1, kRedThreads, 0, s>>>(part.p, grid, part.p + grid);
    count_launch(2);
    TCB_LAUNCH();
    double r = 0;
    d2h(&r, part.p + grid, sizeof(double), s);
    stream_sync(s);
    return r;
}

// max |x| and the finiteness flag of a (small) tensor in one pass and one round
// trip (the quantiser's scale and its non-finite check, core_codec.cpp:55-70)
__global__ void maxfin_stage1(const double* __restrict__ x, u64 n, double* __restrict__ part, int* __restrict__ bad) {
    __shared__ double sh[kRedThreads / 32];
    double m = 0.0;
    bool nonfinite = false;
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double v = x[i];
        nonfinite |= !isfinite(v);
        m = fmax(m, fabs(v));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    if (__syncthreads_or(nonfinite) && threadIdx.x == 0) *bad = 1;
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kRedThreads / 32; ++w) t = fmax(t, sh[w]);
        part[blockIdx.x] = t;
    }
}

double max_abs_finite(const double* x, u64 n, bool* finite, cudaStream_t s) {
    ProfScope prof_scope(kSum, s);
    const int grid = grid_for(n, kRedThreads, 4, 4);
    DevBuf<double> part(grid + 2, s);
    int* bad = reinterpret_cast<int*>(part.p + grid + 1);
    TCB_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    maxfin_stage1<<<grid, kRedThreads, 0, s>>>(x, n, part.p, bad);
    max_stage2<<<1, 1024, 0, s>>>(part.p, grid, part.p + grid);
    count_launch(2);
    TCB_LAUNCH();
    double r[2] = {0, 0};
    d2h(r, part.p + grid, 2 * sizeof(double), s);
    stream_sync(s);
    int b = 0;
    std::memcpy(&b, &r[1], sizeof(int));
    *finite = b == 0;
    return r[0];
}

__global__ void diag_sum_kernel(const double* __restrict__ G, u64 n, double* __restrict__ out) {
    __shared__ double sh[kRedThreads / 32];
    double t = 0.0;
    for (u64 i = threadIdx.x; i < n; i += blockDim.x) t += G[i * n + i];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < kRedThreads / 32; ++w) a += sh[w];
        *out = a;
    }
}

double gram_trace(const double* G, u64 n, cudaStream_t s) {
    DevBuf<double> o(1, s);
    diag_sum_kernel<<<1, kRedThreads, 0, s>>>(G, n, o.p);
    count_launch();
    TCB_LAUNCH();
    return o.to_host()[0];
}

double max_abs(const double* x, u64 n, cudaStream_t s) {
    ProfScope prof_scope(kSum, s);
    const int grid = grid_for(n, kRedThreads, 4, 4);
    DevBuf<double> part(grid + 1, s);
    maxabs_stage1<<<grid, kRedThreads, 0, s>>>(x, n, part.p);
    max_stage2<<<1, 1024, 0, s>>>(part.p, grid, part.p + grid);
    count_launch(2);
    TCB_LAUNCH();
    double r = 0;
    d2h(&r, part.p + grid, sizeof(double), s);
    stream_sync(s);
    return r;
}

template <class T>
void permute_axes(const T* src, T* dst, const std::vector<u64>& shape, const std::vector<u64>& perm,
                  cudaStream_t s) {
    ProfScope prof_scope(kPermute, s);
    const int d = static_cast<int>(shape.size());
    u64 n = 1;
    for (auto v : shape) n *= v;
    bool identity = true;
    for (int i = 0; i < d; ++i) identity &= perm[i] == static_cast<u64>(i);
    if (identity) {
        TCB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
        return;
    }
    if (d == 3 && perm[2] != 2) {
        const u64 nb = shape[perm[2]], na = shape[2];
        const u64 nc = shape[3 - 2 - perm[2]];
        const u64 blocks = ((na + 31) / 32) * ((nb + 31) / 32) * nc;
        permute3_tiled<T><<<static_cast<unsigned>(blocks), dim3(32, 8), 0, s>>>(
            src, dst, shape[0], shape[1], shape[2], static_cast<int>(perm[0]), static_cast<int>(perm[1]),
            static_cast<int>(perm[2]));
        count_launch();
        TCB_LAUNCH();
        return;
    }
    std::vector<u64> st(d);
    u64 acc = 1;
    for (int i = d - 1; i >= 0; --i) {
        st[i] = acc;
        acc *= shape[i];
    }
    std::vector<u64> meta(2 * d);
    for (int i = 0; i < d; ++i) {
        meta[i] = shape[perm[i]];
        meta[d + i] = st[perm[i]];
    }
    DevBuf<u64> m(2 * d, s);
    m.upload(meta.data(), meta.size());
    const unsigned grid = static_cast<unsigned>(sm_count() * 8);
    switch (d) {
        case 1: permute_kernel<T, 1><<<grid, 256, 0, s>>>(src, dst, n, m.p); break;
        case 2: permute_kernel<T, 2><<<grid, 256, 0, s>>>(src, dst, n, m.p); break;
        case 3: permute_kernel<T, 3><<<grid, 256, 0, s>>>(src, dst, n, m.p); break;
        case 4: permute_kernel<T, 4><<<grid, 256, 0, s>>>(src, dst, n, m.p); break;
        case 5: permute_kernel<T, 5><<<grid, 256, 0, s>>>(src, dst, n, m.p); break;
        case 6: permute_kernel<T, 6><<<grid, 256, 0, s>>>(src, dst, n, m.p); break;
        case 7: permute_kernel<T, 7><<<grid, 256, 0, s>>>(src, dst, n, m.p); break;
        case 8: permute_kernel<T, 8><<<grid, 256, 0, s>>>(src, dst, n, m.p); break;
        default: throw Error("transpose: order above 8 unsupported");
    }
    count_launch();
    TCB_LAUNCH();
}
template void permute_axes(const double*, double*, const std::vector<u64>&, const std::vector<u64>&, cudaStream_t);
template void permute_axes(const float*, float*, const std::vector<u64>&, const std::vector<u64>&, cudaStream_t);
template void permute_axes(const u64*, u64*, const std::vector<u64>&, const std::vector<u64>&, cudaStream_t);
template void permute_axes(const u8*, u8*, const std::vector<u64>&, const std::vector<u64>&, cudaStream_t);

}  // namespace tcb
