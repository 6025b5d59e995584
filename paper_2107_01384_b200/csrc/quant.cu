// Core quantisation (core_codec.cpp:55-93), dead slices (:510-523) and the
// Householder sign fold (pipeline.cpp:161-175).  Integer-exact kernels.
#include "kernels.cuh"
#include "quant.cuh"

namespace tcb {

namespace {

// m = nearbyint(ldexp(|x|, k)) (round-half-even), sign = x < 0
__global__ void quantize_kernel(const double* __restrict__ x, u64 n, int k, u64* __restrict__ mag,
                                u8* __restrict__ neg) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double v = x[i];
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
    double s = 0.0;
    for (u64 o = 0; o < outer; ++o) {
        const u64* p = mag + (o * ext + idx) * inner;
        for (u64 q = 0; q < inner; ++q) {
            const double v = __ull2double_rn(p[q]);
            s = __dadd_rn(s, __dmul_rn(v, v));
        }
    }
    out[t] = __dsqrt_rn(__dmul_rn(s, down));
}

__global__ void dead_kernel(const u64* __restrict__ dec, u64 n, const u64* __restrict__ meta /* shape, stride, off */,
                            int d, u8* __restrict__ dead) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 v = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
        if (dec[v] == 0) continue;
        for (int a = 0; a < d; ++a) {
            const u64 idx = (v / meta[d + a]) % meta[a];
            dead[meta[2 * d + a] + idx] = 0;
        }
    }
}

__global__ void signfold_kernel(u8* __restrict__ neg, u64 n, const u64* __restrict__ meta, int d,
                                const signed char* __restrict__ flips /* concatenated per storage axis */) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 v = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
        u8 par = 0;
        for (int a = 0; a < d; ++a) {
            const u64 idx = (v / meta[d + a]) % meta[a];
            par ^= flips[meta[2 * d + a] + idx] < 0 ? 1 : 0;
        }
        neg[v] ^= par;
    }
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

void quantize_f64(const double* x, u64 n, int k, u64* mag, u8* neg, cudaStream_t s) {
    ProfScope prof_scope(kQuant, s);
    if (n == 0) return;
    quantize_kernel<<<sm_count() * 8, 256, 0, s>>>(x, n, k, mag, neg);
    count_launch();
    TCB_LAUNCH();
}

void slice_norms(const u64* mag, const std::vector<u64>& shape, double down, double* out, cudaStream_t s) {
    ProfScope prof_scope(kQuant, s);
    u64 total = 0;
    for (auto v : shape) total += v;
    DevBuf<u64> sh(shape.size(), s);
    sh.upload(shape.data(), shape.size());
    slice_norm_kernel<<<cdiv(total, 64), 64, 0, s>>>(mag, sh.p, static_cast<int>(shape.size()), total, down, out);
    count_launch();
    TCB_LAUNCH();
}

std::vector<u8> dead_slices(const u64* dec, const std::vector<u64>& shape, cudaStream_t s) {
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
    dead_kernel<<<sm_count() * 4, 256, 0, s>>>(dec, n, dm.p, static_cast<int>(shape.size()), dead.p);
    count_launch();
    TCB_LAUNCH();
    return dead.to_host();
}

void sign_fold(u8* neg, const std::vector<u64>& shape, const std::vector<signed char>& flips_by_axis,
               cudaStream_t s) {
    ProfScope prof_scope(kQuant, s);
    const auto meta = axis_meta(shape);
    u64 n = 1;
    for (auto v : shape) n *= v;
    DevBuf<u64> dm(meta.size(), s);
    dm.upload(meta.data(), meta.size());
    DevBuf<signed char> fl(flips_by_axis.size(), s);
    fl.upload(flips_by_axis.data(), flips_by_axis.size());
    signfold_kernel<<<sm_count() * 4, 256, 0, s>>>(neg, n, dm.p, static_cast<int>(shape.size()), fl.p);
    count_launch();
    TCB_LAUNCH();
}

}  // namespace tcb
