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
// One SYRK launch: off-diagonal splits [so0, so0 + off_ctas / n_off) and
// diagonal splits [sd0, sd0 + (grid - off_ctas) / n_diag).  Diagonal tiles
// leave their upper warp blocks idle, so they take per_d = per_o x (active
// warps off / on the diagonal) slabs per CTA: every CTA issues the same DMMA
// count, and the SMs are balanced whatever tiles the scheduler co-locates.
struct SyrkLaunch {
    int n_off, n_diag;
    u64 per_o, per_d, nslab, so0, sd0, splits_o, off_ctas;
};

template <int BK, int ST, int WN>
constexpr int syrk_min_blocks() {  // CTAs per SM the shared memory allows; registers are capped to match
    constexpr int by_smem = (228 * 1024) / (2 * ST * 64 * (BK + 4) * 8 + 1024);
    constexpr int cap = WN == 16 ? 3 : 4;
    return by_smem < 1 ? 1 : (by_smem > cap ? cap : by_smem);
}
// WN: warp tile 32 x WN (16: 8 warps, 8 DMMA per 6 fragment loads; 32: 4 warps,
// 16 independent DMMA per 8 fragment loads).
// One CTA's split-K SYRK over k slabs [s0, s1): ST-stage cp.async ring with
// one barrier per slab; the warp accumulates NS output strips of 32 rows x 8
// columns at (sr[j], sc[j]) of the 64x64 tile (A fragments reloaded only when
// a strip's rows change).  `idle` warps only help load.
template <bool V16, int BK, int ST, int NS>
__device__ __forceinline__ void syrk_run(double (*As)[GT][BK + 4], double (*Bs)[GT][BK + 4],
                                         const double* __restrict__ B, u64 rows, u64 cols, u64 ra, u64 rb, bool diag,
                                         u64 s0, u64 s1, u64 nslab, const int (&sr)[NS], const int (&sc)[NS],
                                         bool idle, double* __restrict__ out) {
    constexpr int PAD = BK + 4;
    const int lane = threadIdx.x & 31;
    const u64 k0 = s0 * BK, k1 = min(cols, s1 * BK);
    double acc[4][NS][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NS; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
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
            double a[4], b[NS];
#pragma unroll
            for (int j = 0; j < NS; ++j) b[j] = Bs_[sc[j] + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int j = 0; j < NS; ++j) {
                if (j == 0 || (NS == 3 && sr[j] != sr[j - 1])) {  // NS 3: diagonal strips change rows
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi) a[mi] = As_[sr[j] + mi * 8 + (lane >> 2)][kk + (lane & 3)];
                }
#pragma unroll
                for (int mi = 0; mi < 4; ++mi) dmma(acc[mi][j][0], acc[mi][j][1], a[mi], b[j]);
            }
        }
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            const int m = sr[j] + mi * 8 + (lane >> 2);
            const int n = sc[j] + 2 * (lane & 3);
            *reinterpret_cast<double2*>(out + m * GT + n) = make_double2(acc[mi][j][0], acc[mi][j][1]);
        }
}

template <bool V16, int BK, int ST, int WN>
__global__ void __launch_bounds__(WN == 16 ? 256 : 128, syrk_min_blocks<BK, ST, WN>()) syrk_kernel(
    const double* __restrict__ B, u64 rows, u64 cols, SyrkLaunch L, double* __restrict__ ws) {
    constexpr int NI = WN / 8, WCOLS = GT / WN;
    constexpr int PAD = BK + 4;
    extern __shared__ __align__(16) double smem_syrk[];
    auto As = reinterpret_cast<double (*)[GT][PAD]>(smem_syrk);
    auto Bs = reinterpret_cast<double (*)[GT][PAD]>(smem_syrk + ST * GT * PAD);
    (void)PAD;
    // CTAs [0, off_ctas): off-diagonal tiles, tile-fastest; then diagonal tiles
    int ti, tj;
    u64 s0, s1;
    double* out;
    if (blockIdx.x < L.off_ctas) {
        const int o = static_cast<int>(blockIdx.x % L.n_off);
        const u64 split = L.so0 + blockIdx.x / L.n_off;
        ti = 1;
        while ((ti + 1) * ti / 2 <= o) ++ti;
        tj = o - ti * (ti - 1) / 2;
        s0 = split * L.per_o;
        s1 = min(L.nslab, s0 + L.per_o);
        out = ws + (split * L.n_off + o) * GT * GT;
    } else {
        const u64 b = blockIdx.x - L.off_ctas;
        const int d = static_cast<int>(b % L.n_diag);
        const u64 split = L.sd0 + b / L.n_diag;
        ti = tj = d;
        s0 = split * L.per_d;
        s1 = min(L.nslab, s0 + L.per_d);
        out = ws + (L.splits_o * L.n_off + split * L.n_diag + d) * GT * GT;
    }
    const int warp = threadIdx.x >> 5;
    const bool diag = ti == tj;
    const u64 ra = static_cast<u64>(ti) * GT, rb = static_cast<u64>(tj) * GT;
    if constexpr (WN == 32) {
        if (diag) {
            // the diagonal tile's 3 lower 32x32 blocks as 12 strips of 32x8,
            // 3 per warp: every warp (so every SM sub-partition) stays busy
            int sr[3], sc[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int idx = 3 * warp + j;
                sr[j] = idx < 4 ? 0 : 32;
                sc[j] = idx < 4 ? 8 * idx : 8 * (idx - 4);
            }
            syrk_run<V16, BK, ST, 3>(As, Bs, B, rows, cols, ra, rb, true, s0, s1, L.nslab, sr, sc, false, out);
            return;
        }
    }
    int sr[NI], sc[NI];
    const int wm = (warp / WCOLS) * 32, wn = (warp % WCOLS) * WN;
#pragma unroll
    for (int j = 0; j < NI; ++j) sr[j] = wm, sc[j] = wn + 8 * j;
    syrk_run<V16, BK, ST, NI>(As, Bs, B, rows, cols, ra, rb, diag, s0, s1, L.nslab, sr, sc,
                              diag && wn >= wm + 32, out);
}

// Kernel shapes (k slab BK, pipeline stages ST); TCB_GRAM_VARIANT picks one
// for measurement, the default is the fastest on the c2 Gram.
struct SyrkVariant {
    int bk, st, threads;
    void (*k16)(const double*, u64, u64, SyrkLaunch, double*);
    void (*k8)(const double*, u64, u64, SyrkLaunch, double*);
    int smem() const { return 2 * st * GT * (bk + 4) * static_cast<int>(sizeof(double)); }
};
#define TCB_SYRK(BK, ST, WN) {BK, ST, WN == 16 ? 256 : 128, syrk_kernel<true, BK, ST, WN>, syrk_kernel<false, BK, ST, WN>}
const SyrkVariant kSyrk[] = {
    TCB_SYRK(32, 2, 16), TCB_SYRK(32, 3, 16), TCB_SYRK(16, 3, 16), TCB_SYRK(16, 4, 16), TCB_SYRK(32, 4, 16),
    TCB_SYRK(32, 2, 32), TCB_SYRK(16, 3, 32), TCB_SYRK(16, 4, 32), TCB_SYRK(32, 3, 32), TCB_SYRK(16, 2, 32),
};
#undef TCB_SYRK
constexpr int kSyrkVariants = sizeof(kSyrk) / sizeof(kSyrk[0]);
constexpr int kSyrkDefault = 6;

// fixed-order split reduction (split 0, 1, ...); writes the full symmetric G (row-major)
__global__ void syrk_reduce(const double* __restrict__ ws, int splits_o, int splits_d, int n_off, int n_diag,
                            u64 rows, double* __restrict__ G) {
    const int tile = blockIdx.x;
    const int e0 = blockIdx.y * (GT * GT / 16), e1 = e0 + GT * GT / 16;
    int ti = 0;
    while ((ti + 1) * (ti + 2) / 2 <= tile) ++ti;
    const int tj = tile - ti * (ti + 1) / 2;
    const bool diag = ti == tj;
    const int splits = diag ? splits_d : splits_o;
    const u64 base = diag ? static_cast<u64>(splits_o) * n_off + ti : static_cast<u64>(ti * (ti - 1) / 2 + tj);
    const u64 stride = diag ? n_diag : n_off;
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const int m = e / GT, n = e % GT;
        const u64 gi = static_cast<u64>(ti) * GT + m, gj = static_cast<u64>(tj) * GT + n;
        if (gi >= rows || gj >= rows || gj > gi) continue;
        // partials fetched 8 at a time (independent loads in flight), summed in split order
        const double* p = ws + base * GT * GT + e;
        const u64 step = stride * GT * GT;
        double s = 0.0;
        int sp = 0;
        for (; sp + 8 <= splits; sp += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = __ldcs(p + (sp + q) * step);
#pragma unroll
            for (int q = 0; q < 8; ++q) s += v[q];
        }
        for (; sp < splits; ++sp) s += __ldcs(p + sp * step);
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

// One CTA computes output tiles (TM columns of B x TN of r) over a range of
// TBK-row k slabs.  Tiles are numbered with the r tile fastest, so the CTAs
// that read the same TM x rows panel of B run together and share it through
// L2 (one DRAM pass over B even when r spans many tiles).  Regular mode: CTA
// b owns tile b, every slab.  Stream-K mode (HBM-bound launches whose tile
// count is close to the resident-CTA count, where the last partial wave would
// idle most SMs): the tiles x slabs units are split evenly over `gridDim.x`
// persistent CTAs; a tile cut into two pieces is summed by two atomic adds
// into the zeroed output (0 + a + b == 0 + b + a: deterministic), which the
// host guarantees by units per CTA >= slabs per tile.
template <bool AV16, int TN>
__global__ void __launch_bounds__(256) ttm_kernel(const double* __restrict__ B, u64 rows, u64 cols,
                                                  const double* __restrict__ U, u64 r, double* __restrict__ out,
                                                  int stream_k) {
    using S = TtmShape<TN>;
    constexpr int MI = S::MI, NI = S::NI, UPAD = S::UPAD;
    extern __shared__ __align__(16) double smem_ttm[];
    auto As = reinterpret_cast<double (*)[TBK][APAD]>(smem_ttm);
    auto Us = reinterpret_cast<double (*)[TBK][UPAD]>(smem_ttm + kTtmStages * TBK * APAD);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = TN == 64 ? (warp >> 1) * 32 : warp * 16, wn = TN == 64 ? (warp & 1) * 32 : 0;
    const u64 nrt = (r + TN - 1) / TN, ntiles = ((cols + TM - 1) / TM) * nrt;
    const int nslab = static_cast<int>((rows + TBK - 1) / TBK);
    u64 u, u_end;  // k-slab units [u, u_end) of tile-major order
    if (stream_k) {
        const u64 units = ntiles * static_cast<u64>(nslab);
        u = units * blockIdx.x / gridDim.x;
        u_end = units * (blockIdx.x + 1) / gridDim.x;
    } else {
        u = static_cast<u64>(blockIdx.x) * nslab;
        u_end = u + nslab;
    }
    while (u < u_end) {
        const u64 tile = u / nslab;
        const int s0 = static_cast<int>(u - tile * nslab);
        const int s1 = static_cast<int>(min(static_cast<u64>(nslab), s0 + (u_end - u)));
        u += static_cast<u64>(s1 - s0);
        const u64 m0 = (tile / nrt) * TM;
        const u64 n0 = (tile % nrt) * TN;
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
        __syncthreads();  // the previous piece's readers are done with every stage
#pragma unroll
        for (int st = 0; st < kTtmStages - 1; ++st) {
            if (s0 + st < s1) load(st, static_cast<u64>(s0 + st) * TBK);
            cp_commit();
        }
        for (int sl = s0; sl < s1; ++sl) {
            const int cur = (sl - s0) % kTtmStages;
            cp_wait<kTtmStages - 2>();
            __syncthreads();
            // refill the stage consumed last iteration (all warps are past it)
            if (sl + kTtmStages - 1 < s1)
                load((sl - s0 + kTtmStages - 1) % kTtmStages, static_cast<u64>(sl + kTtmStages - 1) * TBK);
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
        cp_wait<0>();
        const bool whole = s0 == 0 && s1 == nslab;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
                const u64 m = m0 + wm + mi * 8 + (lane >> 2);
                const u64 n = n0 + wn + ni * 8 + 2 * (lane & 3);
                if (m >= cols) continue;
                if (whole) {
                    if (n < r) out[m * r + n] = acc[mi][ni][0];
                    if (n + 1 < r) out[m * r + n + 1] = acc[mi][ni][1];
                } else {
                    if (n < r) atomicAdd(out + m * r + n, acc[mi][ni][0]);
                    if (n + 1 < r) atomicAdd(out + m * r + n + 1, acc[mi][ni][1]);
                }
            }
    }
}

// ------------------------------------------------------------------ small helpers
// G <- lower triangle mirrored (bitwise symmetric Gram for the eigensolver)
__global__ void mirror_lower_kernel(double* __restrict__ G, u64 n) {
    const u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= n * n) return;
    const u64 i = idx / n, j = idx % n;
    if (j > i) G[idx] = G[j * n + i];
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
    static PerDevice<int> per_sm_dev;
    const int per_sm = per_sm_dev.get([] {
        const SyrkVariant& k = kSyrk[variant];
        cudaFuncSetAttribute(k.k16, cudaFuncAttributeMaxDynamicSharedMemorySize, k.smem());
        cudaFuncSetAttribute(k.k8, cudaFuncAttributeMaxDynamicSharedMemorySize, k.smem());
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k.k16, k.threads, k.smem());
        return std::max(1, b);
    });
    GramPlan gp;
    gp.variant = variant;
    gp.bk = kSyrk[variant].bk;
    const int nt = static_cast<int>((rows + GT - 1) / GT);
    gp.lower = nt * (nt + 1) / 2;
    gp.n_diag = nt;
    gp.n_off = gp.lower - nt;
    gp.nslab = (cols + gp.bk - 1) / gp.bk;
    gp.v16 = (cols % 2 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0);
    // DMMA per warp and k step, off / on the diagonal: 32x32-warp kernels spread
    // a diagonal tile's 3 lower blocks over all 4 warps (16 vs 12).  With
    // TCB_GRAM_DIAG_BALANCE=1 diagonal CTAs take 4/3 the slabs (equal DMMA per
    // CTA); by default every CTA takes the same slabs and the diagonal CTAs'
    // lighter warps leave DMMA issue slots to co-resident CTAs (measured
    // equal or faster on the c2 Gram: profiles/gram_variants_r01.txt).
    static const bool balance = [] {
        const char* e = std::getenv("TCB_GRAM_DIAG_BALANCE");
        return e && *e && *e != '0';
    }();
    const u64 w_o = 4, w_d = (kSyrk[variant].threads == 128 && balance) ? 3 : 4;
    const u64 slots = static_cast<u64>(per_sm) * sm_count();
    auto ctas = [&](u64 po) {
        const u64 pd = (po * w_o + w_d - 1) / w_d;
        return gp.n_off * ((gp.nslab + po - 1) / po) + gp.n_diag * ((gp.nslab + pd - 1) / pd);
    };
    u64 po = std::max<u64>(1, (gp.nslab * (gp.n_off * w_o + gp.n_diag * w_d)) / (w_o * slots));
    while (po < gp.nslab && ctas(po) > slots) ++po;
    gp.per = po;
    gp.per_d = std::min<u64>(gp.nslab, (po * w_o + w_d - 1) / w_d);
    gp.splits = (gp.nslab + gp.per - 1) / gp.per;
    gp.splits_d = (gp.nslab + gp.per_d - 1) / gp.per_d;
    return gp;
}

u64 gram_ws_doubles(const GramPlan& gp) {
    return (gp.splits * gp.n_off + gp.splits_d * gp.n_diag) * GT * GT;
}

u64 gram_split_col(const GramPlan& gp, u64 split, u64 cols) {
    return std::min<u64>(cols, split * gp.per * static_cast<u64>(gp.bk));
}

// Off-diagonal splits [sp0, sp1) plus the diagonal splits whose columns end
// inside (col(sp0), col(sp1)] — every one of them reads only columns below
// col(sp1), and consecutive ranges launch each diagonal split exactly once.
void gram_splits(const double* B, u64 rows, u64 cols, const GramPlan& gp, u64 sp0, u64 sp1, double* ws,
                 cudaStream_t s) {
    if (sp1 <= sp0) return;
    const u64 c0 = gram_split_col(gp, sp0, cols), c1 = sp1 >= gp.splits ? cols : gram_split_col(gp, sp1, cols);
    const u64 dcols = gp.per_d * static_cast<u64>(gp.bk);
    auto dend = [&](u64 d) { return std::min<u64>(cols, (d + 1) * dcols); };
    u64 sd0 = 0;
    if (sp0 > 0)
        while (sd0 < gp.splits_d && dend(sd0) <= c0) ++sd0;
    u64 sd1 = sd0;
    while (sd1 < gp.splits_d && dend(sd1) <= c1) ++sd1;
    ProfScope prof_scope(kGram, s);
    const SyrkVariant& k = kSyrk[gp.variant];
    SyrkLaunch L{gp.n_off, gp.n_diag, gp.per, gp.per_d, gp.nslab, sp0, sd0, gp.splits, (sp1 - sp0) * gp.n_off};
    const unsigned grid = static_cast<unsigned>(L.off_ctas + (sd1 - sd0) * gp.n_diag);
    if (grid == 0) return;
    (gp.v16 ? k.k16 : k.k8)<<<grid, k.threads, k.smem(), s>>>(B, rows, cols, L, ws);
    count_launch();
    TCB_LAUNCH();
}

void gram_reduce(const GramPlan& gp, const double* ws, u64 rows, double* G, cudaStream_t s) {
    ProfScope prof_scope(kGram, s);
    syrk_reduce<<<dim3(gp.lower, 16), 256, 0, s>>>(ws, static_cast<int>(gp.splits), static_cast<int>(gp.splits_d),
                                                   gp.n_off, gp.n_diag, rows, G);
    count_launch();
    TCB_LAUNCH();
}

void gram_f64(const double* B, u64 rows, u64 cols, double* G, cudaStream_t s) {
    const GramPlan gp = gram_plan(B, rows, cols);
    DevBuf<double> ws(gram_ws_doubles(gp), s);
    gram_splits(B, rows, cols, gp, 0, gp.splits, ws.p, s);
    gram_reduce(gp, ws.p, rows, G, s);
}

// Gram of B^T (cols x cols, sthosvd.cpp:91-99 thin branch): B^T B is the TTM of
// B with itself as the factor (DMMA), then mirrored from its lower triangle
void gram_cols_f64(const double* B, u64 rows, u64 cols, double* G, cudaStream_t s) {
    ttm_f64(B, rows, cols, B, cols, G, s);
    ProfScope prof_scope(kGram, s);
    mirror_lower_kernel<<<cdiv(cols * cols, 256), 256, 0, s>>>(G, cols);
    count_launch();
    TCB_LAUNCH();
}

template <int TN>
void launch_ttm(const double* B, u64 rows, u64 cols, const double* U, u64 r, double* out, cudaStream_t s) {
    const u64 ntiles = static_cast<u64>(cdiv(cols, TM)) * cdiv(r, TN);
    const u64 nslab = (rows + TBK - 1) / TBK;
    const bool v16 = (cols % 2 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0);
    constexpr int smem = TtmShape<TN>::smem_doubles * sizeof(double);
    struct Occ {
        int a = 0, b = 0;
    };
    static PerDevice<Occ> occ;
    const Occ& o = occ.get([] {
        Occ x;
        cudaFuncSetAttribute(ttm_kernel<true, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(ttm_kernel<false, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x.a, ttm_kernel<true, TN>, 256, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x.b, ttm_kernel<false, TN>, 256, smem);
        return x;
    });
    // stream-K when the last partial wave would be large and every tile is cut at
    // most once (the HBM-bound small-r projections, e.g. c2's 512 tiles on 444 slots)
    const u64 slots = static_cast<u64>(sm_count()) * static_cast<u64>(std::max(1, v16 ? o.a : o.b));
    const bool sk = TN <= 32 && ntiles > slots && ntiles < 4 * slots && !std::getenv("TCB_TTM_NO_STREAMK");
    const unsigned grid = sk ? static_cast<unsigned>(slots) : static_cast<unsigned>(ntiles);
    if (sk) TCB_CUDA(cudaMemsetAsync(out, 0, cols * r * sizeof(double), s));
    if (v16) ttm_kernel<true, TN><<<grid, 256, smem, s>>>(B, rows, cols, U, r, out, sk ? 1 : 0);
    else ttm_kernel<false, TN><<<grid, 256, smem, s>>>(B, rows, cols, U, r, out, sk ? 1 : 0);
    (void)nslab;
}

void ttm_f64(const double* B, u64 rows, u64 cols, const double* U, u64 r, double* out, cudaStream_t s) {
    ProfScope prof_scope(kTtm, s);
    if (r <= 16) launch_ttm<16>(B, rows, cols, U, r, out, s);
    else if (r <= 32) launch_ttm<32>(B, rows, cols, U, r, out, s);
    else launch_ttm<64>(B, rows, cols, U, r, out, s);
    count_launch();
    TCB_LAUNCH();
}

// out = B V (rows x r): the TTM of B^T (materialised by the tiled permute) with V
void gemm_nn_f64(const double* B, u64 rows, u64 cols, const double* V, u64 r, double* out, cudaStream_t s) {
    DevBuf<double> bt(rows * cols, s);
    permute_axes(B, bt.p, {rows, cols}, {1, 0}, s);
    ttm_f64(bt.p, cols, rows, V, r, out, s);
}

}  // namespace tcb
