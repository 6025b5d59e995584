// Factor codec kernels (factor_codec.cpp:23-149): orthonormality guard,
// Householder reflector extraction as a warp-per-column dataflow (column j
// applies reflectors 0..j-1 as soon as they are published, then publishes its
// own — no grid-wide barriers), the weighted coefficient stream, and the
// decode-side Householder expansion used for the factor error term.
#include <cooperative_groups.h>

#include <cmath>

#include "kernels.cuh"
#include "quant.cuh"

namespace tcb {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// dev[a*rl+b] = |sum_i U_a U_b - delta|, computed in double or float; warp per pair
__global__ void orth_kernel(const double* __restrict__ U, u64 n, u64 r, const u64* __restrict__ live, u64 rl,
                            int as_float, double* __restrict__ dev) {
    const int lane = threadIdx.x & 31;
    const u64 t = static_cast<u64>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (t >= rl * rl) return;
    const u64 a = live[t / rl], b = live[t % rl];
    double out;
    if (as_float) {
        float s = 0.f;
        for (u64 i = lane; i < n; i += 32) s += static_cast<float>(U[i * r + a]) * static_cast<float>(U[i * r + b]);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        out = fabsf(s - (a == b ? 1.f : 0.f));
    } else {
        double s = 0.0;
        for (u64 i = lane; i < n; i += 32) s += U[i * r + a] * U[i * r + b];
        s = warp_sum(s);
        out = fabs(s - (a == b ? 1.0 : 0.0));
    }
    if (lane == 0) dev[t] = out;
}

__global__ void gather_cols(const double* __restrict__ U, u64 n, u64 r, const u64* __restrict__ live, u64 rl,
                            double* __restrict__ R) {
    const u64 t = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n * rl) return;
    const u64 j = t / n, i = t % n;
    R[t] = U[i * r + live[j]];
}

// Warp j owns column j of R (column-major n x rl).  Reflector v_j is published
// to V(:, j) and flag[j] set after a release fence; consumers acquire it.
__global__ void householder_dataflow(double* __restrict__ R, u64 n, u64 rl, double* __restrict__ V,
                                     volatile int* flag, signed char* __restrict__ flips, int* __restrict__ err) {
    const int lane = threadIdx.x & 31;
    const u64 j = static_cast<u64>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (j >= rl) return;
    double* col = R + j * n;
    for (u64 i = 0; i < j; ++i) {
        if (lane == 0)
            while (flag[i] == 0) {
            }
        __syncwarp();
        __threadfence();
        const double* vi = V + i * n;
        double t = 0.0;
        for (u64 k = i + lane; k < n; k += 32) t += __ldcg(vi + k) * col[k];
        t = warp_sum(t);
        for (u64 k = i + lane; k < n; k += 32) col[k] -= 2.0 * t * __ldcg(vi + k);
        __syncwarp();
    }
    // reflector for column j (factor_codec.cpp:34-51)
    double ss = 0.0;
    for (u64 k = j + lane; k < n; k += 32) ss += col[k] * col[k];
    const double nrm = sqrt(warp_sum(ss));
    const double x0 = col[j];
    const double v0 = x0 + (x0 < 0.0 ? -1.0 : 1.0) * nrm;
    double vv = 0.0;
    for (u64 k = j + 1 + lane; k < n; k += 32) vv += col[k] * col[k];
    vv = warp_sum(vv) + v0 * v0;
    const double vn = sqrt(vv);
    if (vn == 0.0) {
        if (lane == 0) *err = 1;
        __threadfence();
        if (lane == 0) flag[j] = 1;
        return;
    }
    // v = (v0, col[j+1:]) / vn ; new R(j,j) = x0 - 2 (v . col) v0
    double dot = 0.0;
    for (u64 k = j + lane; k < n; k += 32) {
        const double vk = (k == j ? v0 : col[k]) / vn;
        dot += vk * col[k];
    }
    dot = warp_sum(dot);
    const double rjj = x0 - 2.0 * dot * (v0 / vn);
    const double sgn = (v0 / vn) < 0.0 ? -1.0 : 1.0;  // canonical positive diagonal
    for (u64 k = lane; k < n; k += 32) {
        double vk = 0.0;
        if (k >= j) vk = sgn * ((k == j ? v0 : col[k]) / vn);
        V[j * n + k] = vk;
    }
    if (lane == 0) flips[j] = rjj < 0.0 ? -1 : 1;
    __threadfence();
    __syncwarp();
    if (lane == 0) flag[j] = 1;
}

__global__ void stream_kernel(const double* __restrict__ V, u64 n, u64 rl, const double* __restrict__ scales,
                              double* __restrict__ st) {
    const u64 j = blockIdx.x;
    if (j >= rl) return;
    const u64 off = j * n - j * (j + 1) / 2;
    for (u64 i = j + 1 + threadIdx.x; i < n; i += blockDim.x) st[off + (i - j - 1)] = V[j * n + i] * scales[j];
}

// decoded stream at candidate plane P[blockIdx.y] -> reflector columns
// (column-major n x rl per plane), diagonal rebuilt from the unit norm
// (factor_codec.cpp:59-77, 119-149).  Fixed-plane decoding: coefficients with
// msb >= P keep planes >= P plus the midpoint (core_codec.cpp:344-367).
__global__ void refl_from_stream(const u64* __restrict__ mag, const u8* __restrict__ neg, int k, u64 n, u64 rl,
                                 const int* __restrict__ planes, const double* __restrict__ scales,
                                 double* __restrict__ Vd, int* __restrict__ err) {
    const int lane = threadIdx.x & 31;
    const u64 j = static_cast<u64>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (j >= rl) return;
    const int P = planes[blockIdx.y];
    double* V = Vd + static_cast<u64>(blockIdx.y) * n * rl;
    const u64 off = j * n - j * (j + 1) / 2;
    double below = 0.0;
    for (u64 i = lane; i < n; i += 32) {
        double v = 0.0;
        if (i > j) {
            const u64 s = off + (i - j - 1);
            const u64 m = mag[s];
            u64 dec = 0;
            if (m != 0 && 63 - __clzll(static_cast<long long>(m)) >= P) {
                dec = (m >> P) << P;
                if (P >= 1) dec += u64{1} << (P - 1);
            }
            double val = scalbn(__ull2double_rn(dec), -k);
            if (neg[s]) val = -val;
            v = val / scales[j];
            below += v * v;
        }
        V[j * n + i] = v;
    }
    below = warp_sum(below);
    if (lane == 0) {
        if (below >= 1.0) *err = 1;
        V[j * n + j] = sqrt(fmax(0.0, 1.0 - below));
    }
}

// X(:, c) = H_0 ... H_{rl-1} e_c ; res[c] = |X(:,c) - flip_c U(:, live_c)|^2.
// Warp per column, NQ entries per lane; reflectors staged CH at a time in smem
// (16, or 8 above 1024 rows: CH n doubles must fit the 227 KB of shared memory).
constexpr int kExChunk = 16;
constexpr u64 kExMaxN = 2304;  // NQ = 72
template <int NQ, int CH = kExChunk>
__global__ void __launch_bounds__(256) expand_residual(const double* __restrict__ Vd, u64 n, u64 rl,
                                                       const double* __restrict__ U, u64 r,
                                                       const u64* __restrict__ live,
                                                       const signed char* __restrict__ flips,
                                                       double* __restrict__ res) {
    extern __shared__ double sv[];
    const int lane = threadIdx.x & 31;
    const u64 c = static_cast<u64>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const double* V = Vd + static_cast<u64>(blockIdx.y) * n * rl;
    const bool active = c < rl;
    double x[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) x[q] = (static_cast<u64>(lane + 32 * q) == c) ? 1.0 : 0.0;
    for (long long hi = static_cast<long long>(rl) - 1; hi >= 0; hi -= CH) {
        const long long lo = hi - CH + 1 < 0 ? 0 : hi - CH + 1;
        __syncthreads();
        for (long long jj = lo; jj <= hi; ++jj)
            for (u64 i = threadIdx.x; i < n; i += blockDim.x) sv[(jj - lo) * n + i] = V[jj * n + i];
        __syncthreads();
        if (!active) continue;
        for (long long jj = hi; jj >= lo; --jj) {
            const double* v = sv + (jj - lo) * n;
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const u64 i = lane + 32 * q;
                if (i >= static_cast<u64>(jj) && i < n) t += v[i] * x[q];
            }
            t = warp_sum(t);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const u64 i = lane + 32 * q;
                if (i >= static_cast<u64>(jj) && i < n) x[q] -= 2.0 * t * v[i];
            }
        }
    }
    if (!active) return;
    const double f = flips[c] < 0 ? -1.0 : 1.0;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const u64 i = lane + 32 * q;
        if (i < n) {
            const double dlt = x[q] - f * U[i * r + live[c]];
            s += dlt * dlt;
        }
    }
    s = warp_sum(s);
    if (lane == 0) res[static_cast<u64>(blockIdx.y) * rl + c] = s;
}

// Decoder side (factor_codec.cpp:246-264): X(:, c) = H_0 ... H_{rl-1} e_c written
// to U(:, live_c) (row-major n x r).  Same warp-per-column expansion as above.
template <int NQ, int CH = kExChunk>
__global__ void __launch_bounds__(256) expand_columns(const double* __restrict__ V, u64 n, u64 rl,
                                                      const u64* __restrict__ live, double* __restrict__ U, u64 r) {
    extern __shared__ double sv[];
    const int lane = threadIdx.x & 31;
    const u64 c = static_cast<u64>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const bool active = c < rl;
    double x[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) x[q] = (static_cast<u64>(lane + 32 * q) == c) ? 1.0 : 0.0;
    for (long long hi = static_cast<long long>(rl) - 1; hi >= 0; hi -= CH) {
        const long long lo = hi - CH + 1 < 0 ? 0 : hi - CH + 1;
        __syncthreads();
        for (long long jj = lo; jj <= hi; ++jj)
            for (u64 i = threadIdx.x; i < n; i += blockDim.x) sv[(jj - lo) * n + i] = V[jj * n + i];
        __syncthreads();
        if (!active) continue;
        for (long long jj = hi; jj >= lo; --jj) {
            const double* v = sv + (jj - lo) * n;
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const u64 i = lane + 32 * q;
                if (i >= static_cast<u64>(jj) && i < n) t += v[i] * x[q];
            }
            t = warp_sum(t);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const u64 i = lane + 32 * q;
                if (i >= static_cast<u64>(jj) && i < n) x[q] -= 2.0 * t * v[i];
            }
        }
    }
    if (!active) return;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const u64 i = lane + 32 * q;
        if (i < n) U[i * r + live[c]] = x[q];
    }
}

}  // namespace

double orth_deviation(const double* U, u64 n, u64 r, const std::vector<u64>& live, bool as_float, cudaStream_t s) {
    ProfScope prof_scope(kFactor, s);
    const u64 rl = live.size();
    if (rl == 0) return 0.0;
    DevBuf<u64> dl(rl, s);
    dl.upload(live.data(), rl);
    DevBuf<double> dev(rl * rl, s);
    orth_kernel<<<cdiv(rl * rl, 8), 256, 0, s>>>(U, n, r, dl.p, rl, as_float ? 1 : 0, dev.p);
    count_launch();
    TCB_LAUNCH();
    const double mx = max_abs(dev.p, rl * rl, s);
    return mx;
}

void householder(const double* U, u64 n, u64 r, const std::vector<u64>& live, double* V, signed char* flips_host,
                 cudaStream_t s) {
    ProfScope prof_scope(kFactor, s);
    const u64 rl = live.size();
    if (rl == 0) return;
    DevBuf<u64> dl(rl, s);
    dl.upload(live.data(), rl);
    DevBuf<double> R(n * rl, s);
    gather_cols<<<cdiv(n * rl, 256), 256, 0, s>>>(U, n, r, dl.p, rl, R.p);
    DevBuf<int> flag(rl + 1, s);
    flag.zero();
    DevBuf<signed char> fl(rl, s);
    DevBuf<int> err(1, s);
    err.zero();
    int nthreads = 256;
    unsigned grid = cdiv(rl, nthreads / 32);
    int maxb = 0;
    TCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, householder_dataflow, nthreads, 0));
    if (static_cast<u64>(maxb) * sm_count() < grid) throw Error("factorize: factor too wide for the dataflow kernel");
    volatile int* fp = flag.p;
    signed char* flp = fl.p;
    int* ep = err.p;
    double* Rp = R.p;
    u64 nn = n, rr = rl;
    void* args[] = {&Rp, &nn, &rr, &V, &fp, &flp, &ep};
    TCB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(householder_dataflow), dim3(grid), dim3(nthreads),
                                         args, 0, s));
    count_launch(2);
    fl.download(flips_host, rl);
    int e = 0;
    err.download(&e, 1);
    stream_sync(s);
    if (e) throw Error("factorize: degenerate reflector");
}

void reflector_stream(const double* V, u64 n, u64 rl, const double* scales_dev, double* st, cudaStream_t s) {
    ProfScope prof_scope(kFactor, s);
    if (rl == 0) return;
    stream_kernel<<<static_cast<unsigned>(rl), 128, 0, s>>>(V, n, rl, scales_dev, st);
    count_launch();
    TCB_LAUNCH();
}

std::vector<double> factor_residuals(const u64* mag, const u8* neg, int k, u64 n, u64 r,
                                     const std::vector<u64>& live, const double* scales_dev, const double* U,
                                     const signed char* flips_dev, const std::vector<int>& planes, cudaStream_t s) {
    ProfScope prof_scope(kFactor, s);
    const u64 rl = live.size();
    const unsigned np = static_cast<unsigned>(planes.size());
    if (n > kExMaxN) throw Error("factor codec: mode sizes above 2304 unsupported on the device path");
    DevBuf<u64> dl(rl, s);
    dl.upload(live.data(), rl);
    DevBuf<int> dp(np, s);
    dp.upload(planes.data(), np);
    DevBuf<double> Vd(n * rl * np, s), res(rl * np, s);
    DevBuf<int> err(1, s);
    err.zero();
    refl_from_stream<<<dim3(cdiv(rl, 4), np), 128, 0, s>>>(mag, neg, k, n, rl, dp.p, scales_dev, Vd.p, err.p);
    const size_t smem = static_cast<size_t>(n <= 1024 ? kExChunk : 8) * n * sizeof(double);
    TCB_ONCE_PER_DEVICE({
        const int mx = kExChunk * 1024 * sizeof(double), mx8 = 8 * static_cast<int>(kExMaxN) * sizeof(double);
        cudaFuncSetAttribute(expand_residual<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(expand_residual<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(expand_residual<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(expand_residual<48, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx8);
        cudaFuncSetAttribute(expand_residual<72, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx8);
    });
    const dim3 grid(cdiv(rl, 8), np);
    if (n <= 256) expand_residual<8><<<grid, 256, smem, s>>>(Vd.p, n, rl, U, r, dl.p, flips_dev, res.p);
    else if (n <= 512) expand_residual<16><<<grid, 256, smem, s>>>(Vd.p, n, rl, U, r, dl.p, flips_dev, res.p);
    else if (n <= 1024) expand_residual<32><<<grid, 256, smem, s>>>(Vd.p, n, rl, U, r, dl.p, flips_dev, res.p);
    else if (n <= 1536) expand_residual<48, 8><<<grid, 256, smem, s>>>(Vd.p, n, rl, U, r, dl.p, flips_dev, res.p);
    else expand_residual<72, 8><<<grid, 256, smem, s>>>(Vd.p, n, rl, U, r, dl.p, flips_dev, res.p);
    count_launch(2);
    TCB_LAUNCH();
    int e = 0;
    err.download(&e, 1);
    auto h = res.to_host();
    if (e) throw Error("reconstruct: reflector sub-diagonal norm reaches 1");
    return h;
}

}  // namespace tcb

namespace tcb {

void factor_expand(const u64* mag, const u8* neg, int k, u64 n, u64 r, const std::vector<u64>& live,
                   const double* scales_dev, double* U, cudaStream_t s, int* err_dev) {
    ProfScope prof_scope(kFactor, s);
    TCB_CUDA(cudaMemsetAsync(U, 0, n * r * sizeof(double), s));
    const u64 rl = live.size();
    if (rl == 0) return;
    if (n > kExMaxN) throw Error("factor codec: mode sizes above 2304 unsupported on the device path");
    DevBuf<u64> dl(rl, s);
    dl.upload(live.data(), rl);
    const int zero = 0;
    DevBuf<int> dp(1, s);
    dp.upload(&zero, 1);
    DevBuf<double> Vd(n * rl, s);
    DevBuf<int> err;
    if (!err_dev) {
        err = DevBuf<int>(1, s);
        err.zero();
    }
    int* ep = err_dev ? err_dev : err.p;
    refl_from_stream<<<dim3(cdiv(rl, 4), 1), 128, 0, s>>>(mag, neg, k, n, rl, dp.p, scales_dev, Vd.p, ep);
    const size_t smem = static_cast<size_t>(n <= 1024 ? kExChunk : 8) * n * sizeof(double);
    TCB_ONCE_PER_DEVICE({
        const int mx = kExChunk * 1024 * sizeof(double), mx8 = 8 * static_cast<int>(kExMaxN) * sizeof(double);
        cudaFuncSetAttribute(expand_columns<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(expand_columns<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(expand_columns<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(expand_columns<48, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx8);
        cudaFuncSetAttribute(expand_columns<72, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx8);
    });
    const unsigned grid = cdiv(rl, 8);
    if (n <= 256) expand_columns<8><<<grid, 256, smem, s>>>(Vd.p, n, rl, dl.p, U, r);
    else if (n <= 512) expand_columns<16><<<grid, 256, smem, s>>>(Vd.p, n, rl, dl.p, U, r);
    else if (n <= 1024) expand_columns<32><<<grid, 256, smem, s>>>(Vd.p, n, rl, dl.p, U, r);
    else if (n <= 1536) expand_columns<48, 8><<<grid, 256, smem, s>>>(Vd.p, n, rl, dl.p, U, r);
    else expand_columns<72, 8><<<grid, 256, smem, s>>>(Vd.p, n, rl, dl.p, U, r);
    count_launch(2);
    TCB_LAUNCH();
    if (err_dev) return;  // the caller checks the shared flag once
    int e = 0;
    err.download(&e, 1);
    stream_sync(s);
    if (e) throw Error("reconstruct: reflector sub-diagonal norm reaches 1");
}

}  // namespace tcb
