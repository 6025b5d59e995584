// Certified top-p eigenpairs of the per-mode Gram (the SelfAdjointEigenSolver
// call of sthosvd.cpp:80-90) for the common low-rank case, without the
// n-step tridiagonalisation:
//
//   Q0 = orth(G W) for a seeded pseudo-random W (n x p), then k rounds of
//   Q <- orth(G Q) (block subspace iteration), then Rayleigh-Ritz:
//   H = Q^T G Q (p x p) -> parallel cyclic Jacobi -> theta, Y; X = Q Y and
//   the residual norms |G x_j - theta_j x_j|.
//
// The host accepts the result only when the rank rule's cutoff falls well
// inside the block and every needed Ritz pair has a residual at the roundoff
// level (then |theta_j - lambda_j| <= |r_j|, and the discarded energy is
// trace(G) - sum theta, at least as accurate as summing the small
// eigenvalues); otherwise it runs the full tridiagonal solver (eig.cu).
//
// orth(): shifted CholQR3 in one CTA -- three Gram / Cholesky / triangular
// solve passes instead of p dependent Householder steps; stable like
// Householder QR (|Z - QR| ~ u |Z|, so a direction's span error is
// u |Z| / sigma_j), which keeps eigenvalues 1e-9 below the largest usable.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "kernels.cuh"

namespace tcb {

namespace {

constexpr int kTkQrThreads = 256;

#ifdef TCB_TOPK_TIMING
__device__ unsigned long long g_tk_phase[32];
#define TK_T(i)                                                     \
    do {                                                            \
        const long long now_ = clock64();                           \
        if (threadIdx.x == 0) atomicAdd(&g_tk_phase[i], now_ - tprev); \
        tprev = now_;                                               \
    } while (0)
#define TK_TC(i)                                                                \
    do {                                                                        \
        const long long now_ = clock64();                                       \
        if (threadIdx.x == 0 && crank == 0) atomicAdd(&g_tk_phase[i], now_ - tprev); \
        tprev = now_;                                                           \
    } while (0)
#else
#define TK_TC(i) \
    do {         \
    } while (0)
#define TK_T(i) \
    do {        \
    } while (0)
#endif
constexpr int kTkRrThreads = 256;

__device__ __forceinline__ double tk_hash_unit(unsigned a, unsigned b) {
    unsigned h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    h *= 0x297A2D39u;
    h ^= h >> 15;
    return (static_cast<double>(h) / 4294967295.0) * 2.0 - 1.0;
}

__device__ __forceinline__ double tk_warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-wide sum with the result broadcast; sh holds 32 doubles
__device__ __forceinline__ double tk_block_sum(double v, double* sh) {
    v = tk_warp_sum(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    const int nw = blockDim.x >> 5;
    for (int w = 0; w < nw; ++w) t += sh[w];
    return t;
}

__global__ void tk_random(double* __restrict__ W, int n, int p) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < n * p) W[idx] = tk_hash_unit(static_cast<unsigned>(idx / p) + 7u, static_cast<unsigned>(idx % p) + 1u);
}

// Shared-memory row stride (doubles) of every n x 32 panel and 32 x 32 matrix:
// 36 = 4 (mod 16), so the DMMA fragment reads below (lane (r, q) = (lane / 4,
// lane % 4) reading element [q][r] or [r][q] of an 8 x 4 / 4 x 8 block) hit 16
// distinct 8-byte banks in each half-warp.
constexpr int kP = 32, kS = 36;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_wait_all() {
    asm volatile("cp.async.commit_group;\n");
    asm volatile("cp.async.wait_group 0;\n");
}

// C (32 x 32, stride kS) = A^T B over rows [0, nr) (nr % 8 == 0) of two staged
// panels, on DMMA: warp w owns the tiles (w / 2, 2 (w % 2) + {0, 1}); two k
// chains per tile for ILP.  diag_add is added to C's diagonal.  8 warps.
__device__ __forceinline__ void tk_atb(const double* A, const double* B, int nr, double* C, double diag_add) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane & 3, r = lane >> 2;
    const int mb = (warp >> 1) * 8, nb = (warp & 1) * 16;
    double c[2][2][2] = {};
    for (int k = 0; k < nr; k += 8) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int kr = (k + 4 * h + q) * kS;
            const double a = A[kr + mb + r];
            const double b0 = B[kr + nb + r], b1 = B[kr + nb + 8 + r];
            dmma(c[h][0][0], c[h][0][1], a, b0);
            dmma(c[h][1][0], c[h][1][1], a, b1);
        }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int row = mb + r, col = nb + 8 * t + 2 * q;
        C[row * kS + col] = (c[0][t][0] + c[1][t][0]) + (row == col ? diag_add : 0.0);
        C[row * kS + col + 1] = (c[0][t][1] + c[1][t][1]) + (row == col + 1 ? diag_add : 0.0);
    }
}

// Z (n x p, row-major) = G (n x n, row-major) W (n x p, row-major) on DMMA.  A
// CTA owns 8 rows of Z; its 8 warps split the k range, each accumulating the
// 8 x 32 block over its k slice from the staged G rows and W, and the 8
// partials are summed in a fixed order.
constexpr int kGqThreads = 256;
__global__ void __launch_bounds__(kGqThreads) tk_gq(const double* __restrict__ G, const double* __restrict__ W, int n,
                                                   int p, double* __restrict__ Z) {
    extern __shared__ __align__(16) double sm_gq[];
    const int nk = (n + 31) & ~31;   // k padded to 8 warps x 4
    const int gs = ((nk + 15) & ~15) + 4;  // G-row stride, = 4 (mod 16)
    double* Gs = sm_gq;                // 8 x gs
    double* Ws = Gs + 8 * gs;          // nk x kS
    double* part = Ws + nk * kS;       // 8 warps x 8 x kS
    const int r0 = blockIdx.x * 8;
    const int nr = min(8, n - r0);
    for (int e = threadIdx.x; e < 8 * nk; e += blockDim.x) {
        const int i = e / nk, k = e % nk;
        if (i < nr && k < n)
            cp_async8(Gs + i * gs + k, G + static_cast<size_t>(r0 + i) * n + k);
        else
            Gs[i * gs + k] = 0.0;
    }
    for (int e = threadIdx.x; e < nk * kP; e += blockDim.x) {
        const int i = e >> 5, j = e & 31;
        if (i < n && j < p)
            cp_async8(Ws + i * kS + j, W + static_cast<size_t>(i) * p + j);
        else
            Ws[i * kS + j] = 0.0;
    }
    cp_wait_all();
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane & 3, r = lane >> 2;
    const int kw = nk / 8, k0 = warp * kw;
    double c[4][2] = {};
    for (int k = k0; k < k0 + kw; k += 4) {
        const double a = Gs[r * gs + k + q];
#pragma unroll
        for (int t = 0; t < 4; ++t) dmma(c[t][0], c[t][1], a, Ws[(k + q) * kS + 8 * t + r]);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        part[(warp * 8 + r) * kS + 8 * t + 2 * q] = c[t][0];
        part[(warp * 8 + r) * kS + 8 * t + 2 * q + 1] = c[t][1];
    }
    __syncthreads();
    const int row = threadIdx.x >> 5, col = threadIdx.x & 31;  // 256 threads = 8 x 32 outputs
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += part[(w * 8 + row) * kS + col];
    if (row < nr && col < p) Z[static_cast<size_t>(r0 + row) * p + col] = v;
}

// 1/sqrt(x) for normal positive x without the range-check branch of rsqrt():
// rsqrt.approx (~2^-20) and one cubic correction step (error ~e^3, measured
// <= 1 ulp on [0.25, 8]).
__device__ __forceinline__ double tk_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(0.375, e, 0.5), y);
}

// C^T-panel products for the column-major panels of tk_cqr: C (32 x 32, stride
// kS) = A^T B with A, B stored transposed (At[m][i] = A[i][m], row stride ld =
// 4 mod 16) over i in [0, nr), nr % 8 == 0.  Same tiling as tk_atb.
__device__ __forceinline__ void tk_atb_t(const double* At, const double* Bt, int ld, int nr, double* C,
                                         double diag_add) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane & 3, r = lane >> 2;
    const int mb = (warp >> 1) * 8, nb = (warp & 1) * 16;
    const double* a_row = At + (mb + r) * ld + q;
    const double* b_row0 = Bt + (nb + r) * ld + q;
    const double* b_row1 = Bt + (nb + 8 + r) * ld + q;
    double c[2][2][2] = {};
    for (int k = 0; k < nr; k += 8) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int kk = k + 4 * h;
            const double a = a_row[kk];
            dmma(c[h][0][0], c[h][0][1], a, b_row0[kk]);
            dmma(c[h][1][0], c[h][1][1], a, b_row1[kk]);
        }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int row = mb + r, col = nb + 8 * t + 2 * q;
        C[row * kS + col] = (c[0][t][0] + c[1][t][0]) + (row == col ? diag_add : 0.0);
        C[row * kS + col + 1] = (c[0][t][1] + c[1][t][1]) + (row == col + 1 ? diag_add : 0.0);
    }
}

// Cholesky of C (32 x 32, stride kS; rows/columns >= p made identity) in its
// elimination form, by the whole CTA with one barrier per column, the same row
// operations also applied to E = I:
//   row_i(C) -= f_i row_k(C),  row_i(E) -= f_i row_k(E),  f_i = C_ki / C_kk  (i > k)
// so E ends as L^-1 for C = L D L^T (L unit lower), and R^-1 = E^T D^-1/2 with
// rinv[k] = D_k^-1/2: T = R^-1 is T[m][c] = E[c][m] rinv[c].  Warp w owns rows
// w, w+8, w+16, w+24, lane j column j; every warp reads the pivot and row k
// itself.  The pivot costs one branch-free rsqrt (1/C_kk = rinv^2), the code
// is compact on purpose: unrolled straight-line variants are instruction-cache
// bound (tools/dbg/chol_lat.cu).  Returns true if a pivot is not a positive
// normal number.
__device__ bool tk_chol_inv(double* C, double* E, double* rinv, int p, int* bad_s) {
    const int j = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int e = threadIdx.x; e < kP * kP; e += blockDim.x) {
        const int i = e >> 5, c = e & 31;
        if (c >= p || i >= p) C[i * kS + c] = i == c ? 1.0 : 0.0;
        E[i * kS + c] = i == c ? 1.0 : 0.0;
    }
    if (threadIdx.x == 0) *bad_s = 0;
    __syncthreads();
#pragma unroll 1
    for (int k = 0; k < kP; ++k) {
        const double dkk = C[k * kS + k];
        const double ckj = C[k * kS + j], ekj = E[k * kS + j];
        double cki[4], cij[4], eij[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = w + 8 * u;
            cki[u] = C[k * kS + i];
            cij[u] = C[i * kS + j];
            eij[u] = E[i * kS + j];
        }
        const bool ok = dkk >= DBL_MIN;
        const double ri = tk_rsqrt(ok ? dkk : 1.0);
        const double inv = ri * ri;
        if (w == 0 && j == 0) {
            rinv[k] = ri;
            if (!ok) *bad_s = 1;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = w + 8 * u;
            if (i > k) {
                const double f = cki[u] * inv;
                C[i * kS + j] = fma(-f, ckj, cij[u]);
                E[i * kS + j] = fma(-f, ekj, eij[u]);
            }
        }
        __syncthreads();
    }
    return *bad_s != 0;
}

// Zt <- (Z T)^T in place for the column-major panel (Zt[m][i] = Z[i][m], stride
// ld) with T = R^-1 from tk_chol_inv, on DMMA: warp w takes the 8-row blocks w,
// w+8, ... of Z; each finishes reading its rows before writing them.
__device__ void tk_apply_inv(double* Zt, int ld, int nr, const double* E, const double* rinv) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane & 3, r = lane >> 2;
    double rc[4];  // rinv of the output columns 8t + r this lane feeds as B
#pragma unroll
    for (int t = 0; t < 4; ++t) rc[t] = rinv[8 * t + r];
    for (int i0 = warp * 8; i0 < nr; i0 += 64) {
        double acc[4][2] = {};
#pragma unroll
        for (int k = 0; k < kP; k += 4) {
            const double a = Zt[(k + q) * ld + i0 + r];  // A[i][m] = Z[i0 + r][k + q]
#pragma unroll
            for (int t = 0; t < 4; ++t)  // B[m][c] = T[k + q][8t + r] = E[8t + r][k + q] rinv[8t + r]
                dmma(acc[t][0], acc[t][1], a, E[(8 * t + r) * kS + k + q] * rc[t]);
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int c = 8 * t + 2 * q;
            Zt[c * ld + i0 + r] = acc[t][0];
            Zt[(c + 1) * ld + i0 + r] = acc[t][1];
        }
    }
}

// Shifted CholQR3 (Fukaya et al. 2020) of Z (n x p row-major, global) -> Q:
// C = Z^T Z + s I (s = 11 (n p + p (p+1)) u |Z|_F^2), Z <- Z R^-1 with R =
// chol(C), then two plain CholQR passes.  The shift bounds cond(Z R^-1) by
// ~u^-1/2, so every Cholesky succeeds for any numerically full-rank block, and
// the result is orthonormal to roundoff (|Z - Q R| ~ u |Z|), like Householder
// QR.  The panel lives column-major in shared memory (row stride = 4 mod 16:
// conflict-free DMMA fragments), p is padded to 32 with zero columns, and the
// Grams and the Z R^-1 products run on DMMA.  *fail is set if a pivot is not
// positive.
__global__ void __launch_bounds__(kTkQrThreads) tk_cqr(const double* __restrict__ Zg, int n, int p,
                                                      double* __restrict__ Q, int* __restrict__ fail) {
    extern __shared__ __align__(16) double sm_tk[];
#ifdef TCB_TOPK_TIMING
    long long tprev = clock64();
#endif
    const int nr = (n + 7) & ~7, ld = ((n + 15) & ~15) + 4;
    double* Zt = sm_tk;          // 32 x ld (columns >= p and rows >= n are zero)
    double* C = Zt + kP * ld;    // 32 x kS: Gram, then eliminated
    double* E = C + kP * kS;     // 32 x kS: L^-1
    double* rinv = E + kP * kS;  // 32
    __shared__ double red[32];
    __shared__ int bad;
    const int tid = threadIdx.x;
    for (int e = tid; e < nr * kP; e += blockDim.x) {
        const int i = e >> 5, j = e & 31;
        if (i < n && j < p)
            cp_async8(Zt + j * ld + i, Zg + static_cast<size_t>(i) * p + j);
        else
            Zt[j * ld + i] = 0.0;
    }
    cp_wait_all();
    __syncthreads();
    double fro = 0.0;
    for (int e = tid; e < n * kP; e += blockDim.x) {
        const double v = Zt[(e / n) * ld + e % n];
        fro = fma(v, v, fro);
    }
    fro = tk_block_sum(fro, red);
    TK_T(0);
    const double shift = 11.0 * (static_cast<double>(n) * p + static_cast<double>(p) * (p + 1)) * (DBL_EPSILON / 2) * fro;
    for (int pass = 0; pass < 3; ++pass) {
        tk_atb_t(Zt, Zt, ld, nr, C, pass == 0 ? shift : 0.0);
        __syncthreads();
        TK_T(1);
        if (tk_chol_inv(C, E, rinv, p, &bad)) break;
        TK_T(2);
        tk_apply_inv(Zt, ld, nr, E, rinv);
        __syncthreads();
        TK_T(3);
    }
    if (bad) {
        if (tid == 0) *fail = 1;
        return;
    }
    for (int e = tid; e < n * p; e += blockDim.x) Q[e] = Zt[(e % p) * ld + e / p];
}

// Jacobi rotation (c, s) annihilating h_ij of the 2 x 2 block [[h_ii, h_ij],
// [h_ij, h_jj]] (smaller angle, sign(s) = sign(h_jj - h_ii) sign(h_ij)), from
// cos 2phi = |a| / hypot(a, b), a = h_jj - h_ii, b = 2 h_ij: two rsqrt on the
// critical path instead of two divides and two square roots.  Branch-free (so
// two rotations interleave): (a, b) are first scaled by an exact power of two
// into [1, 2) by the larger exponent; h_ij = 0 gives the identity.
__device__ __forceinline__ void tk_rotation(double hii, double hjj, double hij, double& c, double& s) {
    const double a = hjj - hii, b = 2.0 * hij;
    const long long em = (__double_as_longlong(fmax(fabs(a), fabs(b))) >> 52) & 0x7ff;
    const long long es = min(max(2046ll - em, 1ll), 2046ll);
    const double sc = __longlong_as_double(es << 52);  // 2^(1023 - em)
    const double as = a * sc, bs = b * sc;
    const double ri = tk_rsqrt(fma(as, as, bs * bs));  // argument in [1, 8)
    const double w = fma(0.5 * fabs(as), ri, 0.5);     // cos^2 phi = (1 + cos 2phi) / 2, in [0.5, 1]
    const double rw = tk_rsqrt(w);
    const bool zero = hij == 0.0;
    c = zero ? 1.0 : w * rw;
    s = zero ? 0.0 : (a >= 0.0 ? 0.5 : -0.5) * bs * ri * rw;  // sin 2phi / (2 cos phi)
}

// Cyclic Jacobi on H (p x p in a 32 x kS buffer) accumulating Y <- Y J, with Y
// stored transposed (Yt[col][row]: a thread's two rows are consecutive across
// the half-warp, so the column updates are bank-conflict free); Hb is a second
// 32 x kS buffer.  256 threads.  Leaves the result in H; returns the number of
// sweeps run.
__device__ int tk_jacobi(double* H, double* Hb, double* Yt, int p, double* red) {
    const int tid = threadIdx.x;
    // Cyclic Jacobi; an odd p gets a dummy player p (its rotations are
    // identities).  One barrier per round: H is double-buffered and the thread
    // owning block (P, Q) computes the rotations of pairs P and Q itself from
    // the previous buffer; it also rotates Y's entries (Q, Q+16) x pair P.
    const int pe = (p + 1) & ~1, half = pe / 2, np1 = pe - 1;
    double* Ha = H;
    auto pair_of = [&](int t, int rnd, int& i, int& j) {
        int x = t - 1 + rnd;
        x = x >= np1 ? x - np1 : x;
        int y = pe - 2 - t + rnd;
        y = y >= np1 ? y - np1 : y;
        i = t == 0 ? 0 : 1 + x;
        j = 1 + y;
        if (i > j) {
            const int tmp = i;
            i = j;
            j = tmp;
        }
    };
    const int P = tid / half, Qp = tid % half;
    const bool active = tid < half * half;
    int sweep = 0;
    for (; sweep < 15; ++sweep) {
        double o = 0.0, d = 0.0;
        for (int a = tid >> 5; a < p; a += blockDim.x >> 5)
            for (int b = tid & 31; b < p; b += 32) {
                const double v = Ha[a * kS + b];
                if (a != b) o = fma(v, v, o);
                else d = fma(v, v, d);
            }
        o = tk_block_sum(o, red);
        d = tk_block_sum(d, red);
        // off(H) <= 1e-14 |diag(H)|: at the roundoff floor (~p eps |H|), after which
        // the eigenvalue error is second order in off(H)
        if (o <= 1e-28 * d) break;
#ifdef TCB_TOPK_TIMING
        if (tid == 0) atomicAdd(&g_tk_phase[8], 1ull);
#endif
        for (int rnd = 0; rnd < np1; ++rnd) {
            if (active) {
                int a0, a1, b0, b1;
                pair_of(P, rnd, a0, a1);
                pair_of(Qp, rnd, b0, b1);
                const bool ra = a1 < p, rb = b1 < p;  // a dummy partner keeps its row/column
                // every load first (indices stay inside the 32 x 32 buffer even for a dummy)
                const double qii = Ha[b0 * kS + b0], qjj = Ha[b1 * kS + b1], qij = Ha[b0 * kS + b1];
                const double h00 = Ha[a0 * kS + b0], h01 = Ha[a0 * kS + b1];
                const double h10 = Ha[a1 * kS + b0], h11 = Ha[a1 * kS + b1];
                const int m0 = Qp, m1 = Qp + 16;  // Y rows of this thread (Y stored transposed)
                const double ya0 = Yt[a0 * kS + m0], yb0 = Yt[a1 * kS + m0];
                const double ya1 = Yt[a0 * kS + m1], yb1 = Yt[a1 * kS + m1];
                // this lane computes pair Q's rotation; pair P's comes from the lane
                // of its half-warp whose Q equals P (half == 16 puts a row P in each half-warp)
                double c2, s2;
                tk_rotation(qii, qjj, qij, c2, s2);
                if (!rb) c2 = 1.0, s2 = 0.0;
                double c1, s1;
                if (half == 16) {
                    const int src = (threadIdx.x & 16) | P;
                    c1 = __shfl_sync(0xffffffffu, c2, src);
                    s1 = __shfl_sync(0xffffffffu, s2, src);
                } else {
                    tk_rotation(Ha[a0 * kS + a0], Ha[a1 * kS + a1], Ha[a0 * kS + a1], c1, s1);
                    if (!ra) c1 = 1.0, s1 = 0.0;
                }
                const double r00 = c1 * h00 - s1 * h10, r01 = c1 * h01 - s1 * h11;
                const double r10 = s1 * h00 + c1 * h10, r11 = s1 * h01 + c1 * h11;
                Hb[a0 * kS + b0] = r00 * c2 - r01 * s2;
                if (rb) Hb[a0 * kS + b1] = r00 * s2 + r01 * c2;
                if (ra) Hb[a1 * kS + b0] = r10 * c2 - r11 * s2;
                if (ra && rb) Hb[a1 * kS + b1] = r10 * s2 + r11 * c2;
                if (ra) {  // Y <- Y J on rows Q, Q+16 (< p) of pair P's columns
                    if (m0 < p) {
                        Yt[a0 * kS + m0] = c1 * ya0 - s1 * yb0;
                        Yt[a1 * kS + m0] = s1 * ya0 + c1 * yb0;
                    }
                    if (m1 < p) {
                        Yt[a0 * kS + m1] = c1 * ya1 - s1 * yb1;
                        Yt[a1 * kS + m1] = s1 * ya1 + c1 * yb1;
                    }
                }
            }
            __syncthreads();
            double* t = Ha;
            Ha = Hb;
            Hb = t;
        }
    }
    if (Ha != H) {  // the current iterate lives in the scratch buffer
        for (int e = tid; e < kP * kP; e += blockDim.x) H[(e >> 5) * kS + (e & 31)] = Ha[(e >> 5) * kS + (e & 31)];
        __syncthreads();
    }
    return sweep;
}

// Rayleigh-Ritz: H = sym(Q^T Z) (Z = G Q) on DMMA, cyclic Jacobi (round-robin
// pairs, every disjoint 2x2 block rotated from both sides in one phase), theta
// descending, then X = Q Y and Z Y on DMMA with the residual norms
// |Z y_j - theta_j x_j| reduced per column in a fixed order, and trace(G).
__global__ void __launch_bounds__(kTkRrThreads) tk_rr(const double* __restrict__ G, const double* __restrict__ Qg,
                                                   const double* __restrict__ Zg, int n, int p,
                                                   double* __restrict__ X, double* __restrict__ out) {
    extern __shared__ __align__(16) double sm_tk[];
#ifdef TCB_TOPK_TIMING
    long long tprev = clock64();
#endif
    const int nr = (n + 7) & ~7;
    double* Qs = sm_tk;            // nr x kS
    double* Zs = Qs + nr * kS;     // nr x kS
    double* H = Zs + nr * kS;      // 32 x kS
    double* Y = H + kP * kS;       // 32 x kS: Q^T Z, then Y transposed (Y[col][row]) during the sweeps
    double* Ys = Y + kP * kS;      // 32 x kS scratch (sorting)
    double* part = Ys + kP * kS;   // 8 warps x 32 residual partials
    __shared__ double red[32];
    __shared__ int order_s[64];
    __shared__ double th_s[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < nr * kP; e += blockDim.x) {
        const int i = e >> 5, j = e & 31;
        if (i < n && j < p) {
            cp_async8(Qs + i * kS + j, Qg + static_cast<size_t>(i) * p + j);
            cp_async8(Zs + i * kS + j, Zg + static_cast<size_t>(i) * p + j);
        } else {
            Qs[i * kS + j] = 0.0;
            Zs[i * kS + j] = 0.0;
        }
    }
    cp_wait_all();
    __syncthreads();
    tk_atb(Qs, Zs, nr, Y, 0.0);  // Y <- Q^T Z
    __syncthreads();
    for (int e = tid; e < kP * kP; e += blockDim.x) {
        const int a = e >> 5, b = e & 31;
        H[a * kS + b] = 0.5 * (Y[a * kS + b] + Y[b * kS + a]);
    }
    __syncthreads();
    for (int e = tid; e < kP * kP; e += blockDim.x) Y[(e >> 5) * kS + (e & 31)] = (e >> 5) == (e & 31) ? 1.0 : 0.0;
    __syncthreads();
    TK_T(4);
    tk_jacobi(H, Ys, Y, p, red);
#ifdef TCB_TOPK_TIMING
    if (tid == 0) atomicAdd(&g_tk_phase[7], 1ull);
#endif
    TK_T(5);
    // theta descending (ties by index)
    if (tid < p) {
        const double t = H[tid * kS + tid];
        int rk = 0;
        for (int q = 0; q < p; ++q) {
            const double u = H[q * kS + q];
            rk += (u > t || (u == t && q < tid)) ? 1 : 0;
        }
        order_s[rk] = tid;
    }
    __syncthreads();
    // Y's columns permuted into descending order (zero beyond p), theta likewise
    for (int e = tid; e < kP * kP; e += blockDim.x) {
        const int m = e >> 5, j = e & 31;
        Ys[m * kS + j] = (m < p && j < p) ? Y[order_s[j] * kS + m] : 0.0;
    }
    if (tid < p) th_s[tid] = H[order_s[tid] * kS + order_s[tid]];
    if (tid >= p && tid < kP) th_s[tid] = 0.0;
    __syncthreads();
    // X = Q Y, W = Z Y on DMMA: warp w takes the 8-row blocks w, w + 8, ...; the
    // residual squares accumulate per (lane, column) in registers, then across
    // the 8 row lanes and the 8 warps in a fixed order.
    {
        const int q = lane & 3, r = lane >> 2;
        double acc[4][2] = {};
        for (int i0 = warp * 8; i0 < nr; i0 += 64) {
            double x[4][2] = {}, w[4][2] = {};
#pragma unroll
            for (int k = 0; k < kP; k += 4) {
                const double aq = Qs[(i0 + r) * kS + k + q], az = Zs[(i0 + r) * kS + k + q];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const double b = Ys[(k + q) * kS + 8 * t + r];
                    dmma(x[t][0], x[t][1], aq, b);
                    dmma(w[t][0], w[t][1], az, b);
                }
            }
            const int i = i0 + r;
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = 8 * t + 2 * q + e;
                    const double rr = w[t][e] - th_s[j] * x[t][e];
                    acc[t][e] = fma(rr, rr, acc[t][e]);  // rows >= n are zero
                    if (i < n && j < p) X[static_cast<size_t>(i) * p + j] = x[t][e];
                }
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                double v = acc[t][e];
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 16);
                if (r == 0) part[warp * kP + 8 * t + 2 * q + e] = v;
            }
    }
    __syncthreads();
    TK_T(6);
    if (tid < p) {
        double s2 = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s2 += part[w * kP + tid];
        out[tid] = th_s[tid];
        out[p + tid] = sqrt(s2);
    }
    double tr = 0.0;
    for (int i = tid; i < n; i += blockDim.x) tr += G[static_cast<size_t>(i) * n + i];
    tr = tk_block_sum(tr, red);
    if (tid == 0) out[2 * p] = tr;
}

// ---------------------------------------------------------------------------
// The whole top-p solve in ONE launch on an 8-CTA thread-block cluster.  CTA c
// owns rows [c nb, c nb + nb) of G (resident in its shared memory for all
// iterations), of Z = G W and of the basis Q; every CTA holds the full current
// basis W (n x 32) for the products.  Per iteration:
//   Z_c = G_c W                       (DMMA, local rows, the flop-heavy part)
//   2 (3 on the last iteration) x { P_c = Z_c^T Z_c (DMMA); cluster barrier; C = sum_c P_c over
//         DSMEM in a fixed order (bitwise identical in every CTA; pass 0 adds
//         the CholQR3 shift from trace C = |Z|_F^2); Cholesky with inverse
//         (redundant per CTA, identical); Z_c <- Z_c R^-1 (DMMA) }
//   all-gather: every CTA stores its rows of Q into every CTA's W (DSMEM);
//   cluster barrier.
// Then Z_c = G_c Q, H = sum_c Q_c^T Z_c, Jacobi (redundant, identical), X_c =
// Q_c Y and the residual/trace partials reduced on CTA 0.  The partial Grams
// are double-buffered, so one cluster barrier per pass suffices.
constexpr int kTkNC = 8;

// C (32 x kS) = A^T B over nr rows (nr % 8 == 0) of row-major panels, for
// remote-free local use (same tiling as tk_atb).
__device__ __forceinline__ void tk_cl_gq(const double* Gl, int gs, const double* W, int nk, int nb, double* Zl) {
    // Zl (nb x 32, stride kS) = Gl (nb x nk, stride gs) W (nk x 32, stride kS);
    // warp w: row block w & 3, column tiles 2 (w >> 2) + {0, 1}; two k chains
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane & 3, r = lane >> 2;
    const int rb = (warp & 3) * 8, t0 = (warp >> 2) * 2;
    if (rb >= nb) return;
    double c[2][2][2] = {};
    const double* a_row = Gl + (rb + r) * gs + q;
    for (int k = 0; k < nk; k += 8) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int kk = k + 4 * h;
            const double a = a_row[kk];
            const double* b = W + (kk + q) * kS + r;
            dmma(c[h][0][0], c[h][0][1], a, b[8 * t0]);
            dmma(c[h][1][0], c[h][1][1], a, b[8 * (t0 + 1)]);
        }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int col = 8 * (t0 + t) + 2 * q;
        Zl[(rb + r) * kS + col] = c[0][t][0] + c[1][t][0];
        Zl[(rb + r) * kS + col + 1] = c[0][t][1] + c[1][t][1];
    }
}

// Zl (nb x 32 row-major) <- Zl T, T = R^-1 (E, rinv): results held in
// registers across a CTA barrier (warps w and w + 4 share row block w & 3)
__device__ __forceinline__ void tk_cl_apply(double* Zl, int nb, const double* E, const double* rinv) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane & 3, r = lane >> 2;
    const int rb = (warp & 3) * 8, t0 = (warp >> 2) * 2;
    double acc[2][2] = {};
    if (rb < nb) {
        const double rc0 = rinv[8 * t0 + r], rc1 = rinv[8 * (t0 + 1) + r];
#pragma unroll
        for (int k = 0; k < kP; k += 4) {
            const double a = Zl[(rb + r) * kS + k + q];
            dmma(acc[0][0], acc[0][1], a, E[(8 * t0 + r) * kS + k + q] * rc0);
            dmma(acc[1][0], acc[1][1], a, E[(8 * (t0 + 1) + r) * kS + k + q] * rc1);
        }
    }
    __syncthreads();
    if (rb < nb) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int col = 8 * (t0 + t) + 2 * q;
            Zl[(rb + r) * kS + col] = acc[t][0];
            Zl[(rb + r) * kS + col + 1] = acc[t][1];
        }
    }
}

__global__ void __launch_bounds__(256) tk_cluster(const double* __restrict__ G, int n, int p, int iters,
                                                  double* __restrict__ X, double* __restrict__ out) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double sm_cl[];
    const int crank = static_cast<int>(cl.block_rank());
    const int nk = (n + 31) & ~31, gs = ((nk + 15) & ~15) + 4;
    const int nb = (((n + kTkNC - 1) / kTkNC) + 7) & ~7;
    const int nw = max(nk, kTkNC * nb);
    const int r0 = crank * nb, nl = max(0, min(n, r0 + nb) - r0);
    double* Gl = sm_cl;               // nb x gs: rows [r0, r0 + nl) of G, zero padded
    double* W = Gl + nb * gs;         // nw x kS: the full basis (rows >= n zero)
    double* Zl = W + nw * kS;         // nb x kS
    double* Pg = Zl + nb * kS;        // 2 x 32 x kS: partial Grams (double-buffered, read remotely)
    double* C = Pg + 2 * kP * kS;     // 32 x kS
    double* E = C + kP * kS;          // 32 x kS
    double* Ys = E + kP * kS;         // 32 x kS (Rayleigh-Ritz)
    double* rinv = Ys + kP * kS;      // 32
    double* part = rinv + kP;         // kTkNC x (2 kP + 1): residual / trace partials (CTA 0's is used)
    __shared__ double red[32];
    __shared__ int bad;
    __shared__ int order_s[64];
    __shared__ double th_s[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef TCB_TOPK_TIMING
    long long tprev = clock64();
#endif
    // ---- load the owned rows of G, generate W (the same seeded hash as tk_random)
    for (int e = tid; e < nb * nk; e += blockDim.x) {
        const int i = e / nk, k = e % nk;
        if (i < nl && k < n)
            cp_async8(Gl + i * gs + k, G + static_cast<size_t>(r0 + i) * n + k);
        else
            Gl[i * gs + k] = 0.0;
    }
    for (int e = tid; e < nw * kP; e += blockDim.x) {
        const int i = e >> 5, j = e & 31;
        W[i * kS + j] = (i < n && j < p) ? tk_hash_unit(static_cast<unsigned>(i) + 7u, static_cast<unsigned>(j) + 1u)
                                         : 0.0;
    }
    if (tid == 0) bad = 0;
    cp_wait_all();
    __syncthreads();
    TK_TC(16);
    int pb = 0;  // partial-Gram buffer toggle
    auto reduce_pg = [&](double* dst) {  // dst = sum over the cluster of Pg[pb], fixed order
        for (int e = tid; e < kP * kP; e += blockDim.x) {
            const int off = pb * kP * kS + (e >> 5) * kS + (e & 31);
            double v = 0.0;
#pragma unroll
            for (int c = 0; c < kTkNC; ++c) v += cl.map_shared_rank(Pg, c)[off];
            dst[(e >> 5) * kS + (e & 31)] = v;
        }
    };
    for (int it = 0; it < iters; ++it) {
        tk_cl_gq(Gl, gs, W, nk, nb, Zl);
        __syncthreads();
        TK_TC(17);
        // intermediate iterations only need the span (the next product is
        // re-orthonormalised): shifted CholQR2 there, the full CholQR3 on the
        // basis the Rayleigh-Ritz step uses
        const int passes = it == iters - 1 ? 3 : 2;
        for (int pass = 0; pass < passes; ++pass) {
            tk_atb(Zl, Zl, nb, Pg + pb * kP * kS, 0.0);
            TK_TC(18);
            cl.sync();
            TK_TC(19);
            reduce_pg(C);
            __syncthreads();
            TK_TC(20);
            if (pass == 0) {  // CholQR3 shift from |Z|_F^2 = trace C (identical in every CTA)
                double tr = 0.0;
                for (int j = 0; j < p; ++j) tr += C[j * kS + j];
                const double shift =
                    11.0 * (static_cast<double>(n) * p + static_cast<double>(p) * (p + 1)) * (DBL_EPSILON / 2) * tr;
                __syncthreads();
                if (tid < p) C[tid * kS + tid] += shift;
            }
            pb ^= 1;
            if (tk_chol_inv(C, E, rinv, p, &bad)) break;
            TK_TC(21);
            tk_cl_apply(Zl, nb, E, rinv);
            __syncthreads();
            TK_TC(22);
        }
        if (bad) break;  // identical in every CTA
        // all-gather the new basis rows into every CTA's W
        for (int e = tid; e < nl * kP; e += blockDim.x) {
            const int i = e >> 5, j = e & 31;
            const double v = j < p ? Zl[i * kS + j] : 0.0;
#pragma unroll
            for (int c = 0; c < kTkNC; ++c) cl.map_shared_rank(W, c)[(r0 + i) * kS + j] = v;
        }
        TK_TC(23);
        cl.sync();
        TK_TC(24);
    }
    if (bad) {
        if (crank == 0 && tid == 0) reinterpret_cast<int*>(out + 2 * p + 1)[0] = 1;
        cl.sync();
        return;
    }
    // ---- Rayleigh-Ritz: Z = G Q, H = sym(Q^T Z) over the cluster
    tk_cl_gq(Gl, gs, W, nk, nb, Zl);
    __syncthreads();
    tk_atb(W + r0 * kS, Zl, nb, Pg + pb * kP * kS, 0.0);  // local Q rows (zero beyond n)
    cl.sync();
    reduce_pg(E);  // E <- Q^T Z
    __syncthreads();
    double* H = C;
    for (int e = tid; e < kP * kP; e += blockDim.x) {
        const int a = e >> 5, b = e & 31;
        H[a * kS + b] = 0.5 * (E[a * kS + b] + E[b * kS + a]);
    }
    __syncthreads();
    double* Yt = E;
    for (int e = tid; e < kP * kP; e += blockDim.x) Yt[(e >> 5) * kS + (e & 31)] = (e >> 5) == (e & 31) ? 1.0 : 0.0;
    __syncthreads();
    TK_TC(25);
    tk_jacobi(H, Ys, Yt, p, red);
    TK_TC(26);
    if (tid < p) {
        const double t = H[tid * kS + tid];
        int rk = 0;
        for (int q = 0; q < p; ++q) {
            const double u = H[q * kS + q];
            rk += (u > t || (u == t && q < tid)) ? 1 : 0;
        }
        order_s[rk] = tid;
    }
    __syncthreads();
    for (int e = tid; e < kP * kP; e += blockDim.x) {
        const int m = e >> 5, j = e & 31;
        Ys[m * kS + j] = (m < p && j < p) ? Yt[order_s[j] * kS + m] : 0.0;
    }
    if (tid < p) th_s[tid] = H[order_s[tid] * kS + order_s[tid]];
    if (tid >= p && tid < kP) th_s[tid] = 0.0;
    __syncthreads();
    // X_c = Q_c Y, R_c = Z_c Y - X_c diag(theta): warp w row block w & 3, column tiles 2 (w >> 2) + {0, 1}
    double* wpart = Pg + (pb ^ 1) * kP * kS;  // 8 warps x 32 columns (that buffer is no longer read remotely)
    {
        const int q = lane & 3, r = lane >> 2;
        const int rb = (warp & 3) * 8, t0 = (warp >> 2) * 2;
        double x[2][2] = {}, w2[2][2] = {};
        if (rb < nb) {
#pragma unroll
            for (int k = 0; k < kP; k += 4) {
                const double aq = W[(r0 + rb + r) * kS + k + q], az = Zl[(rb + r) * kS + k + q];
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const double b = Ys[(k + q) * kS + 8 * (t0 + t) + r];
                    dmma(x[t][0], x[t][1], aq, b);
                    dmma(w2[t][0], w2[t][1], az, b);
                }
            }
        }
        const int i = rb + r;
        double acc[2][2];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int j = 8 * (t0 + t) + 2 * q + e;
                const double rr = w2[t][e] - th_s[j] * x[t][e];
                acc[t][e] = (rb < nb && i < nl) ? rr * rr : 0.0;
                if (rb < nb && i < nl && j < p) X[static_cast<size_t>(r0 + i) * p + j] = x[t][e];
            }
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                double v = acc[t][e];
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 16);
                if (r == 0) wpart[warp * kP + 8 * (t0 + t) + 2 * q + e] = v;
            }
    }
    __syncthreads();
    // CTA partials (fixed warp order: warps w and w + 4 cover the same columns of different tiles)
    double* dst0 = cl.map_shared_rank(part, 0) + crank * (2 * kP + 1);
    if (tid < kP) {
        double s2 = 0.0;
        for (int w = 0; w < 8; ++w) s2 += ((w >> 2) * 16 <= tid && tid < (w >> 2) * 16 + 16) ? wpart[w * kP + tid] : 0.0;
        dst0[tid] = s2;
    }
    double tr = 0.0;
    for (int i = tid; i < nl; i += blockDim.x) tr += Gl[i * gs + r0 + i];
    tr = tk_block_sum(tr, red);
    if (tid == 0) dst0[2 * kP] = tr;
    cl.sync();
    if (crank == 0 && tid < p) {
        double s2 = 0.0;
        for (int c = 0; c < kTkNC; ++c) s2 += part[c * (2 * kP + 1) + tid];
        out[tid] = th_s[tid];
        out[p + tid] = sqrt(s2);
    }
    if (crank == 0 && tid == 0) {
        double t = 0.0;
        for (int c = 0; c < kTkNC; ++c) t += part[c * (2 * kP + 1) + 2 * kP];
        out[2 * p] = t;
    }
    TK_TC(27);
}

}  // namespace

#ifdef TCB_TOPK_TIMING
void topk_phase_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_tk_phase, sizeof(unsigned long long) * 32); }
#endif

bool cholqr_inplace(double* U, u64 n64, int r, int* fail_dev, cudaStream_t s) {
    if (n64 > 256 || r < 1 || r > kP || n64 < static_cast<u64>(r)) return false;
    TCB_ONCE_PER_DEVICE(cudaFuncSetAttribute(tk_cqr, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    TCB_CUDA(cudaMemsetAsync(fail_dev, 0, sizeof(int), s));
    const size_t qld = ((n64 + 15) & ~u64{15}) + 4;
    const size_t qsm = (kP * qld + 2 * kP * kS + kP) * sizeof(double);
    tk_cqr<<<1, kTkQrThreads, qsm, s>>>(U, static_cast<int>(n64), r, U, fail_dev);
    count_launch();
    TCB_LAUNCH();
    return true;
}

bool topk_supported(u64 n, int p) {  // shared-memory footprints: tk_rr (3 n p + 2 p^2) and tk_gq (n (p + 8))
    return p >= 8 && p <= 32 && n >= static_cast<u64>(2 * p) && n <= 256;
}

void topk_eig(const double* G, u64 n64, int p, int extra_iters, double* X, std::vector<double>& theta,
              std::vector<double>& resid, double& trace, cudaStream_t s) {
    ProfScope prof_scope(kEig, s);
    const int n = static_cast<int>(n64);
    TCB_ONCE_PER_DEVICE({
        cudaFuncSetAttribute(tk_gq, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(tk_cqr, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(tk_rr, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    });
    DevBuf<double> out(2 * p + 2, s);
    TCB_CUDA(cudaMemsetAsync(out.p, 0, (2 * p + 2) * sizeof(double), s));
    // one launch on an 8-CTA cluster when it fits (the multi-launch path below otherwise)
    {
        const int nk = (n + 31) & ~31, gs = ((nk + 15) & ~15) + 4;
        const int nb = (((n + kTkNC - 1) / kTkNC) + 7) & ~7, nw = std::max(nk, kTkNC * nb);
        const size_t smem = (static_cast<size_t>(nb) * gs + static_cast<size_t>(nw) * kS + nb * kS + 5 * kP * kS +
                             kP + kTkNC * (2 * kP + 1)) * sizeof(double);
        static PerDevice<bool> cl_attr_dev;
        const bool cl_attr = cl_attr_dev.get([] {
            return cudaFuncSetAttribute(tk_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024) ==
                   cudaSuccess;
        });
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kTkNC);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = kTkNC;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        static PerDevice<int> ncl_dev;
        const int ncl = ncl_dev.get([&] {
            int v = 0;
            if (!cl_attr || cudaOccupancyMaxActiveClusters(&v, tk_cluster, &cfg) != cudaSuccess) v = 0;
            cudaGetLastError();
            return v;
        });
        const char* e = std::getenv("TCB_TOPK_NO_CLUSTER");
        if (ncl > 0 && smem <= 224 * 1024 && !(e && *e && *e != '0')) {
            TCB_CUDA(cudaLaunchKernelEx(&cfg, tk_cluster, G, n, p, extra_iters + 1, X, out.p));
            count_launch(1);
            TCB_LAUNCH();
            std::vector<double> h(2 * p + 2);
            out.download(h.data(), 2 * p + 2);
            stream_sync(s);
            int failed = 0;
            std::memcpy(&failed, &h[2 * p + 1], sizeof(int));
            if (failed) {
                theta.assign(p, 0.0);
                resid.assign(p, HUGE_VAL);
                trace = 0.0;
                return;
            }
            theta.assign(h.begin(), h.begin() + p);
            resid.assign(h.begin() + p, h.begin() + 2 * p);
            trace = h[2 * p];
            return;
        }
    }
    DevBuf<double> W(n64 * p, s), Z(n64 * p, s);
    int* fail = reinterpret_cast<int*>(out.p + 2 * p + 1);
    tk_random<<<cdiv(n64 * p, 256), 256, 0, s>>>(W.p, n, p);
    const size_t nr = (n64 + 7) & ~u64{7}, nk = (n64 + 31) & ~u64{31}, gs = ((nk + 15) & ~u64{15}) + 4;
    const size_t gsm = (8 * gs + nk * kS + 64 * kS) * sizeof(double);
    const size_t qld = ((n64 + 15) & ~u64{15}) + 4;
    const size_t qsm = (kP * qld + 2 * kP * kS + kP) * sizeof(double);
    const size_t rsm = (2 * nr * kS + 3 * kP * kS + 8 * kP) * sizeof(double);
    for (int it = 0; it <= extra_iters; ++it) {
        tk_gq<<<cdiv(n64, 8), kGqThreads, gsm, s>>>(G, W.p, n, p, Z.p);
        tk_cqr<<<1, kTkQrThreads, qsm, s>>>(Z.p, n, p, W.p, fail);
    }
    tk_gq<<<cdiv(n64, 8), kGqThreads, gsm, s>>>(G, W.p, n, p, Z.p);
    tk_rr<<<1, kTkRrThreads, rsm, s>>>(G, W.p, Z.p, n, p, X, out.p);
    count_launch(2 * (extra_iters + 1) + 3);
    TCB_LAUNCH();
    std::vector<double> h(2 * p + 2);
    out.download(h.data(), 2 * p + 2);
    stream_sync(s);
    int failed = 0;
    std::memcpy(&failed, &h[2 * p + 1], sizeof(int));
    if (failed) {  // a Cholesky pivot broke down: report "not converged"
        theta.assign(p, 0.0);
        resid.assign(p, HUGE_VAL);
        trace = 0.0;
        return;
    }
    theta.assign(h.begin(), h.begin() + p);
    resid.assign(h.begin() + p, h.begin() + 2 * p);
    trace = h[2 * p];
}

}  // namespace tcb
