// fp64 tensor-core contractions of the ST-HOSVD mode loop (sthosvd.cpp:72-99,158-166).
//
//  * gram_f64 : G = B B^T  (SYRK, lower-triangle 64x64 tiles, deterministic split-K)
//  * ttm_f64  : out = B^T U (the projection fused with the circular mode shift)
//
// Both use DMMA (mma.sync.m8n8k4.f64 — tcgen05 has no f64 kind on sm_100a) fed
// by cp.async double-buffered shared-memory tiles with bank-conflict-free
// padding.  Split-K partials are reduced in a fixed order, so results are
// bitwise reproducible run to run.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace tcb {

namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ------------------------------------------------------------------ SYRK
constexpr int GT = 64;  // output tile

// Load rows [r0, r0+64) x k [k0, k0+BK) of row-major B into s[64][BK+4]
// (row stride BK+4 doubles: the fragment reads below are bank-conflict free).
template <bool V16, int BK>
__device__ __forceinline__ void load_slab(double (*s)[BK + 4], const double* __restrict__ B, u64 rows, u64 cols,
                                          u64 r0, u64 k0, u64 k1) {
    if constexpr (V16) {
        // 64 rows x BK/2 chunks of 16 B
        for (int c = threadIdx.x; c < GT * (BK / 2); c += blockDim.x) {
            const int rr = c / (BK / 2), kk = (c % (BK / 2)) * 2;
            const u64 gr = r0 + rr, gk = k0 + kk;
            const bool ok = gr < rows && gk < k1;  // k1 even here: pairs never straddle
            cp_async16(&s[rr][kk], ok ? B + gr * cols + gk : B, ok);
        }
    } else {
        for (int c = threadIdx.x; c < GT * BK; c += blockDim.x) {
            const int rr = c / BK, kk = c % BK;
            const u64 gr = r0 + rr, gk = k0 + kk;
            const bool ok = gr < rows && gk < k1;
            cp_async8(&s[rr][kk], ok ? B + gr * cols + gk : B, ok);
        }
    }
}

// Split-K SYRK sized to the machine: grid = tiles x splits with splits =
// floor(SMs x resident CTAs / tiles), so every SM gets the same DMMA work
// (a fixed split count leaves SMs with 2 or 3 CTAs), and blockIdx runs tile-
// fastest so the CTAs resident together cover all lower-triangle tiles of the
// same k-chunk and share B's row blocks through L2 (one DRAM pass over B).
// ST-stage cp.async ring with one barrier per k slab.  On a diagonal tile the
// two warps whose 32x16 block lies wholly above the diagonal issue no DMMA
// (the reduction never reads the upper half): 10 % less tensor work on a
// 256-row Gram, which co-resident CTAs' warps pick up.
template <int BK, int ST, int WN>
constexpr int syrk_min_blocks() {  // CTAs per SM the shared memory allows; registers are capped to match
    constexpr int by_smem = (228 * 1024) / (2 * ST * 64 * (BK + 4) * 8 + 1024);
    constexpr int cap = WN == 16 ? 3 : 4;
    return by_smem < 1 ? 1 : (by_smem > cap ? cap : by_smem);
}
// WN: warp tile 32 x WN (16: 8 warps, 8 DMMA per 6 fragment loads; 32: 4 warps,
// 16 independent DMMA per 8 fragment loads).
template <bool V16, int BK, int ST, int WN>
__global__ void __launch_bounds__(WN == 16 ? 256 : 128, syrk_min_blocks<BK, ST, WN>()) syrk_kernel(
    const double* __restrict__ B, u64 rows, u64 cols, int ntiles_lower, u64 slabs_per_split, u64 nslab, u64 split0,
    double* __restrict__ ws) {
    constexpr int NI = WN / 8, WCOLS = GT / WN;
    constexpr int PAD = BK + 4;
    extern __shared__ __align__(16) double smem_syrk[];
    auto As = reinterpret_cast<double (*)[GT][PAD]>(smem_syrk);
    auto Bs = reinterpret_cast<double (*)[GT][PAD]>(smem_syrk + ST * GT * PAD);
    const int tile = blockIdx.x % ntiles_lower;
    const u64 split = split0 + blockIdx.x / ntiles_lower;
    const u64 s0 = split * slabs_per_split, s1 = min(nslab, s0 + slabs_per_split);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp / WCOLS) * 32, wn = (warp % WCOLS) * WN;
    int ti = 0;
    while ((ti + 1) * (ti + 2) / 2 <= tile) ++ti;
    const int tj = tile - ti * (ti + 1) / 2;
    const bool diag = ti == tj;
    const bool idle = diag && wn >= wm + 32;
    const u64 k0 = s0 * BK, k1 = min(cols, s1 * BK);
    const u64 ra = static_cast<u64>(ti) * GT, rb = static_cast<u64>(tj) * GT;
    double acc[4][NI][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int ns = s1 > s0 ? static_cast<int>(s1 - s0) : 0;
    auto load = [&](int buf, int sl) {
        const u64 kn = k0 + static_cast<u64>(sl) * BK;
        load_slab<V16, BK>(As[buf], B, rows, cols, ra, kn, k1);
        if (!diag) load_slab<V16, BK>(Bs[buf], B, rows, cols, rb, kn, k1);
    };
#pragma unroll
    for (int st = 0; st < ST - 1; ++st) {
        if (st < ns) load(st, st);
        cp_commit();
    }
    for (int sl = 0; sl < ns; ++sl) {
        const int cur = sl % ST;
        cp_wait<ST - 2>();
        __syncthreads();
        // refill the stage consumed last iteration (every warp is past it)
        if (sl + ST - 1 < ns) load((sl + ST - 1) % ST, sl + ST - 1);
        cp_commit();
        if (idle) continue;
        double (*As_)[PAD] = As[cur];
        double (*Bs_)[PAD] = diag ? As[cur] : Bs[cur];
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[4], b[NI];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = As_[wm + mi * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) b[ni] = Bs_[wn + ni * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
    }
    double* out = ws + (split * ntiles_lower + tile) * GT * GT;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
            const int m = wm + mi * 8 + (lane >> 2);
            const int n = wn + ni * 8 + 2 * (lane & 3);
            *reinterpret_cast<double2*>(out + m * GT + n) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
        }
}

// Kernel shapes (k slab BK, pipeline stages ST); TCB_GRAM_VARIANT picks one
// for measurement, the default is the fastest on the c2 Gram.
struct SyrkVariant {
    int bk, st, threads;
    void (*k16)(const double*, u64, u64, int, u64, u64, u64, double*);
    void (*k8)(const double*, u64, u64, int, u64, u64, u64, double*);
    int smem() const { return 2 * st * GT * (bk + 4) * static_cast<int>(sizeof(double)); }
};
#define TCB_SYRK(BK, ST, WN) {BK, ST, WN == 16 ? 256 : 128, syrk_kernel<true, BK, ST, WN>, syrk_kernel<false, BK, ST, WN>}
const SyrkVariant kSyrk[] = {
    TCB_SYRK(32, 2, 16), TCB_SYRK(32, 3, 16), TCB_SYRK(16, 3, 16), TCB_SYRK(16, 4, 16), TCB_SYRK(32, 4, 16),
    TCB_SYRK(32, 2, 32), TCB_SYRK(16, 3, 32), TCB_SYRK(16, 4, 32), TCB_SYRK(32, 3, 32), TCB_SYRK(16, 2, 32),
};
#undef TCB_SYRK
constexpr int kSyrkVariants = sizeof(kSyrk) / sizeof(kSyrk[0]);
constexpr int kSyrkDefault = 7;

// fixed-order split reduction (split 0, 1, ...); writes the full symmetric G (row-major)
__global__ void syrk_reduce(const double* __restrict__ ws, int splits, int ntiles_lower, u64 rows,
                            double* __restrict__ G) {
    const int tile = blockIdx.x;
    const int e0 = blockIdx.y * (GT * GT / 16), e1 = e0 + GT * GT / 16;
    int ti = 0;
    while ((ti + 1) * (ti + 2) / 2 <= tile) ++ti;
    const int tj = tile - ti * (ti + 1) / 2;
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const int m = e / GT, n = e % GT;
        const u64 gi = static_cast<u64>(ti) * GT + m, gj = static_cast<u64>(tj) * GT + n;
        if (gi >= rows || gj >= rows || gj > gi) continue;
        double s = 0.0;
        for (int sp = 0; sp < splits; ++sp) s += ws[(static_cast<u64>(sp) * ntiles_lower + tile) * GT * GT + e];
        G[gi * rows + gj] = s;
        G[gj * rows + gi] = s;
    }
}

// ------------------------------------------------------------------ TTM
// out (cols x r) = B^T U: HBM-bound for small r (one pass over B), so the
// output tile width follows r (TN = 16 / 32 / 64) instead of padding every
// projection to 64 columns of DMMA work, and B streams through a 3-stage
// cp.async pipeline (TM = 128 columns of B x TBK = 16 rows per stage).
constexpr int TM = 128, TBK = 16, kTtmStages = 3;
constexpr int APAD = TM + 4;

template <int TN>
struct TtmShape {  // 8 warps: TN 64 -> 4x2 warps of 32x32; else 8x1 warps of 16 x TN
    static constexpr int WM = TN == 64 ? 32 : 16, WN = TN == 64 ? 32 : TN;
    static constexpr int MI = WM / 8, NI = WN / 8, UPAD = TN + 4;
    static constexpr int smem_doubles = kTtmStages * TBK * (APAD + UPAD);
};

template <bool AV16, int TN>
__global__ void __launch_bounds__(256) ttm_kernel(const double* __restrict__ B, u64 rows, u64 cols,
                                                  const double* __restrict__ U, u64 r, double* __restrict__ out) {
    using S = TtmShape<TN>;
    constexpr int MI = S::MI, NI = S::NI, UPAD = S::UPAD;
    extern __shared__ __align__(16) double smem_ttm[];
    auto As = reinterpret_cast<double (*)[TBK][APAD]>(smem_ttm);
    auto Us = reinterpret_cast<double (*)[TBK][UPAD]>(smem_ttm + kTtmStages * TBK * APAD);
    const u64 m0 = static_cast<u64>(blockIdx.x) * TM;
    const u64 n0 = static_cast<u64>(blockIdx.y) * TN;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = TN == 64 ? (warp >> 1) * 32 : warp * 16, wn = TN == 64 ? (warp & 1) * 32 : 0;
    double acc[MI][NI][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    auto load = [&](int buf, u64 k0) {
        if constexpr (AV16) {
            for (int c = threadIdx.x; c < TBK * (TM / 2); c += blockDim.x) {
                const int kk = c / (TM / 2), mm = (c % (TM / 2)) * 2;
                const u64 gk = k0 + kk, gm = m0 + mm;
                const bool ok = gk < rows && gm < cols;  // cols even: pairs never straddle
                cp_async16(&As[buf][kk][mm], ok ? B + gk * cols + gm : B, ok);
            }
        } else {
            for (int c = threadIdx.x; c < TBK * TM; c += blockDim.x) {
                const int kk = c / TM, mm = c % TM;
                const u64 gk = k0 + kk, gm = m0 + mm;
                const bool ok = gk < rows && gm < cols;
                cp_async8(&As[buf][kk][mm], ok ? B + gk * cols + gm : B, ok);
            }
        }
        for (int c = threadIdx.x; c < TBK * TN; c += blockDim.x) {
            const int kk = c / TN, nn = c % TN;
            const u64 gk = k0 + kk, gn = n0 + nn;
            const bool ok = gk < rows && gn < r;
            cp_async8(&Us[buf][kk][nn], ok ? U + gk * r + gn : U, ok);
        }
    };
    const int nslab = static_cast<int>((rows + TBK - 1) / TBK);
#pragma unroll
    for (int st = 0; st < kTtmStages - 1; ++st) {
        if (st < nslab) load(st, static_cast<u64>(st) * TBK);
        cp_commit();
    }
    for (int sl = 0; sl < nslab; ++sl) {
        const int cur = sl % kTtmStages;
        cp_wait<kTtmStages - 2>();
        __syncthreads();
        // refill the stage consumed last iteration (all warps are past it)
        if (sl + kTtmStages - 1 < nslab) load((sl + kTtmStages - 1) % kTtmStages, static_cast<u64>(sl + kTtmStages - 1) * TBK);
        cp_commit();
#pragma unroll
        for (int kk = 0; kk < TBK; kk += 4) {
            double a[MI], b[NI];
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) a[mi] = As[cur][kk + (lane & 3)][wm + mi * 8 + (lane >> 2)];
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) b[ni] = Us[cur][kk + (lane & 3)][wn + ni * 8 + (lane >> 2)];
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
    }
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
            const u64 m = m0 + wm + mi * 8 + (lane >> 2);
            const u64 n = n0 + wn + ni * 8 + 2 * (lane & 3);
            if (m >= cols) continue;
            if (n < r) out[m * r + n] = acc[mi][ni][0];
            if (n + 1 < r) out[m * r + n + 1] = acc[mi][ni][1];
        }
}

// ------------------------------------------------------------------ small helpers
__global__ void gram_cols_kernel(const double* __restrict__ B, u64 rows, u64 cols, double* __restrict__ G) {
    const u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= cols * cols) return;
    const u64 i = idx / cols, j = idx % cols;
    if (j > i) return;
    double s = 0.0;
    for (u64 k = 0; k < rows; ++k) s = fma(B[k * cols + i], B[k * cols + j], s);
    G[i * cols + j] = s;
    G[j * cols + i] = s;
}

__global__ void gemm_nn_kernel(const double* __restrict__ B, u64 rows, u64 cols, const double* __restrict__ V, u64 r,
                               double* __restrict__ out) {
    const u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= rows * r) return;
    const u64 i = idx / r, j = idx % r;
    double s = 0.0;
    for (u64 k = 0; k < cols; ++k) s = fma(B[i * cols + k], V[k * r + j], s);
    out[idx] = s;
}

// Peak probe: independent DMMA chains per warp, no memory traffic.
__global__ void dmma_peak_kernel(int iters, double* out) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

}  // namespace

double peak_dmma_tflops() {
    cudaStream_t s = nullptr;
    DevBuf<double> o(1, s);
    const int iters = 4096, blocks = sm_count() * 4, threads = 256;
    dmma_peak_kernel<<<blocks, threads, 0, s>>>(64, o.p);  // warm-up
    cudaEvent_t a, b;
    TCB_CUDA(cudaEventCreate(&a));
    TCB_CUDA(cudaEventCreate(&b));
    TCB_CUDA(cudaEventRecord(a, s));
    dmma_peak_kernel<<<blocks, threads, 0, s>>>(iters, o.p);
    TCB_CUDA(cudaEventRecord(b, s));
    TCB_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    TCB_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (static_cast<double>(blocks) * threads / 32);
    return flops / (ms * 1e-3) / 1e12;
}

GramPlan gram_plan(const double* B, u64 rows, u64 cols) {
    static const int variant = [] {
        const char* e = std::getenv("TCB_GRAM_VARIANT");
        const int v = e && *e ? std::atoi(e) : kSyrkDefault;
        return v >= 0 && v < kSyrkVariants ? v : kSyrkDefault;
    }();
    static const int per_sm = [] {
        const SyrkVariant& k = kSyrk[variant];
        cudaFuncSetAttribute(k.k16, cudaFuncAttributeMaxDynamicSharedMemorySize, k.smem());
        cudaFuncSetAttribute(k.k8, cudaFuncAttributeMaxDynamicSharedMemorySize, k.smem());
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k.k16, k.threads, k.smem());
        return std::max(1, b);
    }();
    GramPlan gp;
    gp.variant = variant;
    gp.bk = kSyrk[variant].bk;
    const int nt = static_cast<int>((rows + GT - 1) / GT);
    gp.lower = nt * (nt + 1) / 2;
    gp.nslab = (cols + gp.bk - 1) / gp.bk;
    gp.v16 = (cols % 2 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0);
    const u64 slots = static_cast<u64>(per_sm) * sm_count();
    u64 splits = std::max<u64>(1, std::min<u64>(gp.nslab, slots / gp.lower));
    gp.per = (gp.nslab + splits - 1) / splits;
    gp.splits = (gp.nslab + gp.per - 1) / gp.per;
    return gp;
}

u64 gram_ws_doubles(const GramPlan& gp) { return gp.splits * gp.lower * GT * GT; }

u64 gram_split_col(const GramPlan& gp, u64 split, u64 cols) {
    return std::min<u64>(cols, split * gp.per * static_cast<u64>(gp.bk));
}

void gram_splits(const double* B, u64 rows, u64 cols, const GramPlan& gp, u64 sp0, u64 sp1, double* ws,
                 cudaStream_t s) {
    if (sp1 <= sp0) return;
    ProfScope prof_scope(kGram, s);
    const SyrkVariant& k = kSyrk[gp.variant];
    const unsigned grid = static_cast<unsigned>((sp1 - sp0) * gp.lower);
    (gp.v16 ? k.k16 : k.k8)<<<grid, k.threads, k.smem(), s>>>(B, rows, cols, gp.lower, gp.per, gp.nslab, sp0, ws);
    count_launch();
    TCB_LAUNCH();
}

void gram_reduce(const GramPlan& gp, const double* ws, u64 rows, double* G, cudaStream_t s) {
    ProfScope prof_scope(kGram, s);
    syrk_reduce<<<dim3(gp.lower, 16), 256, 0, s>>>(ws, static_cast<int>(gp.splits), gp.lower, rows, G);
    count_launch();
    TCB_LAUNCH();
}

void gram_f64(const double* B, u64 rows, u64 cols, double* G, cudaStream_t s) {
    const GramPlan gp = gram_plan(B, rows, cols);
    DevBuf<double> ws(gram_ws_doubles(gp), s);
    gram_splits(B, rows, cols, gp, 0, gp.splits, ws.p, s);
    gram_reduce(gp, ws.p, rows, G, s);
}

void gram_cols_f64(const double* B, u64 rows, u64 cols, double* G, cudaStream_t s) {
    ProfScope prof_scope(kGram, s);
    gram_cols_kernel<<<cdiv(cols * cols, 256), 256, 0, s>>>(B, rows, cols, G);
    count_launch();
    TCB_LAUNCH();
}

template <int TN>
void launch_ttm(const double* B, u64 rows, u64 cols, const double* U, u64 r, double* out, cudaStream_t s) {
    dim3 grid(cdiv(cols, TM), cdiv(r, TN));
    const bool v16 = (cols % 2 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0);
    constexpr int smem = TtmShape<TN>::smem_doubles * sizeof(double);
    static bool attr = [] {
        cudaFuncSetAttribute(ttm_kernel<true, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(ttm_kernel<false, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        return true;
    }();
    (void)attr;
    if (v16) ttm_kernel<true, TN><<<grid, 256, smem, s>>>(B, rows, cols, U, r, out);
    else ttm_kernel<false, TN><<<grid, 256, smem, s>>>(B, rows, cols, U, r, out);
}

void ttm_f64(const double* B, u64 rows, u64 cols, const double* U, u64 r, double* out, cudaStream_t s) {
    ProfScope prof_scope(kTtm, s);
    if (r <= 16) launch_ttm<16>(B, rows, cols, U, r, out, s);
    else if (r <= 32) launch_ttm<32>(B, rows, cols, U, r, out, s);
    else launch_ttm<64>(B, rows, cols, U, r, out, s);
    count_launch();
    TCB_LAUNCH();
}

void gemm_nn_f64(const double* B, u64 rows, u64 cols, const double* V, u64 r, double* out, cudaStream_t s) {
    ProfScope prof_scope(kTtm, s);
    gemm_nn_kernel<<<cdiv(rows * r, 256), 256, 0, s>>>(B, rows, cols, V, r, out);
    count_launch();
    TCB_LAUNCH();
}

}  // namespace tcb
