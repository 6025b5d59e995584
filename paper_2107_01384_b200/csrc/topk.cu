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
#include <cfloat>
#include <cmath>
#include <cstring>

#include "kernels.cuh"

namespace tcb {

namespace {

constexpr int kTkQrThreads = 256;

#ifdef TCB_TOPK_TIMING
__device__ unsigned long long g_tk_phase[16];
#define TK_T(i)                                                     \
    do {                                                            \
        const long long now_ = clock64();                           \
        if (threadIdx.x == 0) atomicAdd(&g_tk_phase[i], now_ - tprev); \
        tprev = now_;                                               \
    } while (0)
#else
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

// Z (n x p, row-major) = G (n x n, row-major) Q (n x p, row-major).  A CTA owns
// 8 rows of Z: it stages those 8 rows of G and all of Q in shared memory
// (coalesced), then thread (row, col) runs its dot product from shared memory.
__global__ void __launch_bounds__(256) tk_gq(const double* __restrict__ G, const double* __restrict__ Q, int n, int p,
                                            double* __restrict__ Z) {
    extern __shared__ double sm_gq[];
    double* Gs = sm_gq;       // 8 x n
    double* Qs = Gs + 8 * n;  // n x p
    const int r0 = blockIdx.x * 8;
    const int nr = min(8, n - r0);
    for (int idx = threadIdx.x; idx < nr * n; idx += blockDim.x) Gs[idx] = G[static_cast<size_t>(r0) * n + idx];
    for (int idx = threadIdx.x; idx < n * p; idx += blockDim.x) Qs[idx] = Q[idx];
    __syncthreads();
    for (int o = threadIdx.x; o < nr * p; o += blockDim.x) {
        const int r = o / p, c = o % p;
        const double* g = Gs + r * n;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int k = 0;
        for (; k + 4 <= n; k += 4) {
            a0 = fma(g[k], Qs[k * p + c], a0);
            a1 = fma(g[k + 1], Qs[(k + 1) * p + c], a1);
            a2 = fma(g[k + 2], Qs[(k + 2) * p + c], a2);
            a3 = fma(g[k + 3], Qs[(k + 3) * p + c], a3);
        }
        for (; k < n; ++k) a0 = fma(g[k], Qs[k * p + c], a0);
        Z[static_cast<size_t>(r0 + r) * p + c] = (a0 + a1) + (a2 + a3);
    }
}

// Block-parallel Cholesky of C (32 x 33 shared; p <= 32 real columns, the rest
// made identity): C = R^T R, R (upper) written to a separate 32 x 33 array so
// one barrier per column suffices (the trailing update reads the unscaled row
// k of C while row k of R is written).  Returns true if a pivot is not positive.
__device__ bool tk_block_chol(double* C, double* R, int p, int* bad_s) {
    constexpr int P = 32, PP = 33;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < P * P; e += nt) {
        const int i = e >> 5, j = e & 31;
        if (j >= p) C[i * PP + j] = i == j ? 1.0 : 0.0;
        R[i * PP + j] = 0.0;
    }
    if (tid == 0) *bad_s = 0;
    __syncthreads();
    for (int k = 0; k < P; ++k) {
        const double dkk = C[k * PP + k];
        const double inv = dkk > 0.0 ? 1.0 / dkk : 0.0;
        if (tid < P && tid >= k) {
            const double r = sqrt(dkk > 0.0 ? dkk : 1.0);
            R[k * PP + tid] = tid == k ? r : C[k * PP + tid] / r;
        }
        if (tid == 0 && !(dkk > 0.0)) *bad_s = 1;
        for (int e = tid; e < P * P; e += nt) {  // trailing update, k < i <= j, from the unscaled row k
            const int i = e >> 5, j = e & 31;
            if (i > k && j >= i) C[i * PP + j] = fma(-C[k * PP + i] * inv, C[k * PP + j], C[i * PP + j]);
        }
        __syncthreads();
    }
    return *bad_s != 0;
}

// Z row <- Z row R^-1 for every row (thread per row), column sweep with the
// row in registers: z_m /= R_mm, then z_j -= z_m R_mj for all j > m (independent FMAs)
__device__ void tk_rows_solve(double* Zs, int n, const double* C) {
    constexpr int P = 32, PP = 33;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double z[P];
#pragma unroll
        for (int m = 0; m < P; ++m) z[m] = Zs[i * PP + m];
#pragma unroll
        for (int m = 0; m < P; ++m) {
            z[m] = z[m] / C[m * PP + m];
#pragma unroll
            for (int j = m + 1; j < P; ++j) z[j] = fma(-z[m], C[m * PP + j], z[j]);
        }
#pragma unroll
        for (int m = 0; m < P; ++m) Zs[i * PP + m] = z[m];
    }
}

// Shifted CholQR3 (Fukaya et al. 2020) of Z (n x p row-major, global) -> Q:
// C = Z^T Z + s I (s = 11 (n p + p (p+1)) u |Z|_F^2), R = chol(C), Z <- Z R^-1,
// then two plain CholQR passes.  The shift bounds cond(Z R^-1) by ~u^-1/2, so
// every Cholesky succeeds for any numerically full-rank block, and the result
// is orthonormal to roundoff with |Z - Q R| ~ u |Z|, like Householder QR.
// p is padded to 32 (identity columns); one warp factors C and inverts R in
// registers (lane j owns column j), the rest is register-blocked for ILP.
// *fail is set if a pivot is not positive.
__global__ void __launch_bounds__(kTkQrThreads) tk_cqr(const double* __restrict__ Zg, int n, int p,
                                                      double* __restrict__ Q, int* __restrict__ fail) {
    extern __shared__ double sm_tk[];
#ifdef TCB_TOPK_TIMING
    long long tprev = clock64();
#endif
    constexpr int P = 32, PP = 33;
    double* Zs = sm_tk;        // n x PP (columns >= p are zero)
    double* C = Zs + n * PP;   // P x PP: Gram
    double* R = C + P * PP;    // P x PP: Cholesky factor (upper)
    __shared__ double red[32];
    __shared__ int bad;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    double fro = 0.0;
    for (int i = warp; i < n; i += nw) {
        const double v = lane < p ? Zg[static_cast<size_t>(i) * p + lane] : 0.0;
        Zs[i * PP + lane] = v;
        fro = fma(v, v, fro);
    }
    if (tid == 0) bad = 0;
    fro = tk_block_sum(fro, red);
    TK_T(0);
    const double shift = 11.0 * (static_cast<double>(n) * p + static_cast<double>(p) * (p + 1)) * (DBL_EPSILON / 2) * fro;
    const int a0 = (tid >> 4) * 2, b0 = (tid & 15) * 2;  // this thread's 2x2 block of C (256 threads)
    for (int pass = 0; pass < 3; ++pass) {
        if (tid < 256) {
            double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
#pragma unroll 4
            for (int i = 0; i < n; ++i) {
                const double za0 = Zs[i * PP + a0], za1 = Zs[i * PP + a0 + 1];
                const double zb0 = Zs[i * PP + b0], zb1 = Zs[i * PP + b0 + 1];
                c00 = fma(za0, zb0, c00);
                c01 = fma(za0, zb1, c01);
                c10 = fma(za1, zb0, c10);
                c11 = fma(za1, zb1, c11);
            }
            const double sh = pass == 0 ? shift : 0.0;
            C[a0 * PP + b0] = c00 + (a0 == b0 ? sh : 0.0);
            C[a0 * PP + b0 + 1] = c01;
            C[(a0 + 1) * PP + b0] = c10;
            C[(a0 + 1) * PP + b0 + 1] = c11 + (a0 == b0 ? sh : 0.0);
        }
        __syncthreads();
        TK_T(1);
        if (tk_block_chol(C, R, p, &bad)) break;
        TK_T(2);
        tk_rows_solve(Zs, n, R);
        __syncthreads();
        TK_T(3);
    }
    if (bad) {
        if (tid == 0) *fail = 1;
        return;
    }
    for (int i = warp; i < n; i += nw)
        if (lane < p) Q[static_cast<size_t>(i) * p + lane] = Zs[i * PP + lane];
}

// Rayleigh-Ritz: H = Q^T Z (Z = G Q), cyclic Jacobi (round-robin pairs, every
// disjoint 2x2 block rotated from both sides in one phase), theta descending,
// X = Q Y, residual norms |Z y_j - theta_j x_j|, and trace(G).
__global__ void __launch_bounds__(kTkRrThreads) tk_rr(const double* __restrict__ G, const double* __restrict__ Qg,
                                                   const double* __restrict__ Zg, int n, int p,
                                                   double* __restrict__ X, double* __restrict__ out) {
    extern __shared__ double sm_tk[];
#ifdef TCB_TOPK_TIMING
    long long tprev = clock64();
#endif
    const int pp = p + 1;
    double* Qs = sm_tk;           // n x pp
    double* Zs = Qs + n * pp;     // n x pp
    double* H = Zs + n * pp;      // p x pp
    double* Y = H + p * pp;       // p x pp (Y[row][col])
    double* R2 = Y + p * pp;      // p x n residual squares
    __shared__ double red[32];
    __shared__ double cs[32][2];
    __shared__ int pr[32][2];
    __shared__ int order_s[64];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int i = warp; i < n; i += nw)
        if (lane < p) {
            Qs[i * pp + lane] = Qg[static_cast<size_t>(i) * p + lane];
            Zs[i * pp + lane] = Zg[static_cast<size_t>(i) * p + lane];
        }
    __syncthreads();
    // H = sym(Q^T Z): thread (a0, b0) owns a 2x2 block (p <= 32, 256 threads)
    {
        const int a0 = (tid >> 4) * 2, b0 = (tid & 15) * 2;
        if (a0 < p && b0 < p) {
            const bool a1 = a0 + 1 < p, b1 = b0 + 1 < p;
            double qz00 = 0.0, qz01 = 0.0, qz10 = 0.0, qz11 = 0.0, zq00 = 0.0, zq01 = 0.0, zq10 = 0.0, zq11 = 0.0;
#pragma unroll 4
            for (int i = 0; i < n; ++i) {
                const double* qi = Qs + i * pp;
                const double* zi = Zs + i * pp;
                const double qa0 = qi[a0], qa1 = a1 ? qi[a0 + 1] : 0.0, qb0 = qi[b0], qb1 = b1 ? qi[b0 + 1] : 0.0;
                const double za0 = zi[a0], za1 = a1 ? zi[a0 + 1] : 0.0, zb0 = zi[b0], zb1 = b1 ? zi[b0 + 1] : 0.0;
                qz00 = fma(qa0, zb0, qz00);
                qz01 = fma(qa0, zb1, qz01);
                qz10 = fma(qa1, zb0, qz10);
                qz11 = fma(qa1, zb1, qz11);
                zq00 = fma(za0, qb0, zq00);
                zq01 = fma(za0, qb1, zq01);
                zq10 = fma(za1, qb0, zq10);
                zq11 = fma(za1, qb1, zq11);
            }
            H[a0 * pp + b0] = 0.5 * (qz00 + zq00);
            if (b1) H[a0 * pp + b0 + 1] = 0.5 * (qz01 + zq01);
            if (a1) H[(a0 + 1) * pp + b0] = 0.5 * (qz10 + zq10);
            if (a1 && b1) H[(a0 + 1) * pp + b0 + 1] = 0.5 * (qz11 + zq11);
        }
    }
    for (int e = tid; e < p * p; e += blockDim.x) Y[(e / p) * pp + e % p] = (e / p == e % p) ? 1.0 : 0.0;
    __syncthreads();
    TK_T(4);
    // cyclic Jacobi; an odd p gets a dummy player p (its rotations are identities)
    const int pe = (p + 1) & ~1, half = pe / 2;
    for (int sweep = 0; sweep < 15; ++sweep) {
        double o = 0.0, d = 0.0;
        for (int a = tid >> 5; a < p; a += blockDim.x >> 5)
            for (int b = tid & 31; b < p; b += 32) {
                const double v = H[a * pp + b];
                if (a != b) o = fma(v, v, o);
                else d = fma(v, v, d);
            }
        o = tk_block_sum(o, red);
        d = tk_block_sum(d, red);
        // off(H) <= 1e-14 |diag(H)|: at the roundoff floor (~p eps |H|), after which
        // the eigenvalue error is second order in off(H)
        if (o <= 1e-28 * d) break;
        for (int rnd = 0; rnd < pe - 1; ++rnd) {
            if (tid < half) {  // pair t and its rotation
                const int t = tid;
                int i = t == 0 ? 0 : 1 + (t - 1 + rnd) % (pe - 1);
                int j = 1 + (pe - 2 - t + rnd) % (pe - 1);
                if (i > j) {
                    const int tmp = i;
                    i = j;
                    j = tmp;
                }
                double c = 1.0, s = 0.0;
                if (j < p) {
                    const double hij = H[i * pp + j];
                    if (hij != 0.0) {
                        const double th = (H[j * pp + j] - H[i * pp + i]) / (2.0 * hij);
                        const double tt = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(fma(th, th, 1.0)));
                        c = 1.0 / sqrt(fma(tt, tt, 1.0));
                        s = tt * c;
                    }
                }
                cs[t][0] = c;
                cs[t][1] = s;
                pr[t][0] = i;
                pr[t][1] = j;
            }
            __syncthreads();
            // H <- J^T H J on every 2x2 block (pair P rows, pair Q cols)
            for (int e = tid; e < half * half; e += blockDim.x) {
                const int P = e / half, Qp = e % half;
                const int a0 = pr[P][0], a1 = pr[P][1], b0 = pr[Qp][0], b1 = pr[Qp][1];
                const double c1 = cs[P][0], s1 = cs[P][1], c2 = cs[Qp][0], s2 = cs[Qp][1];
                const bool ra = a1 < p, rb = b1 < p;  // a dummy partner keeps its row/column
                const double h00 = H[a0 * pp + b0], h01 = rb ? H[a0 * pp + b1] : 0.0;
                const double h10 = ra ? H[a1 * pp + b0] : 0.0, h11 = (ra && rb) ? H[a1 * pp + b1] : 0.0;
                const double r00 = c1 * h00 - s1 * h10, r01 = c1 * h01 - s1 * h11;
                const double r10 = s1 * h00 + c1 * h10, r11 = s1 * h01 + c1 * h11;
                H[a0 * pp + b0] = r00 * c2 - r01 * s2;
                if (rb) H[a0 * pp + b1] = r00 * s2 + r01 * c2;
                if (ra) H[a1 * pp + b0] = r10 * c2 - r11 * s2;
                if (ra && rb) H[a1 * pp + b1] = r10 * s2 + r11 * c2;
            }
            // Y <- Y J
            for (int e = tid; e < p * half; e += blockDim.x) {
                const int m = e / half, P = e % half;
                const int a = pr[P][0], b = pr[P][1];
                if (b >= p) continue;
                const double c = cs[P][0], s = cs[P][1];
                const double ya = Y[m * pp + a], yb = Y[m * pp + b];
                Y[m * pp + a] = c * ya - s * yb;
                Y[m * pp + b] = s * ya + c * yb;
            }
            __syncthreads();
        }
    }
    TK_T(5);
    // theta descending (ties by index)
    if (tid < p) {
        const double t = H[tid * pp + tid];
        int rk = 0;
        for (int q = 0; q < p; ++q) {
            const double u = H[q * pp + q];
            rk += (u > t || (u == t && q < tid)) ? 1 : 0;
        }
        order_s[rk] = tid;
    }
    __syncthreads();
    // Y and theta permuted into descending order (R2 doubles as scratch until the residuals)
    double* Ys = R2;  // p x pp scratch, free until the residual squares are written below
    double* th_s = Ys + p * pp;
    for (int e = tid; e < p * p; e += blockDim.x) {
        const int m = e / p, j = e % p;
        Ys[m * pp + j] = Y[m * pp + order_s[j]];
    }
    if (tid < p) th_s[tid] = H[order_s[tid] * pp + order_s[tid]];
    __syncthreads();
    for (int e = tid; e < p * p; e += blockDim.x) Y[(e / p) * pp + e % p] = Ys[(e / p) * pp + e % p];
    if (tid < p) H[tid * pp + tid] = th_s[tid];  // H's diagonal now holds theta in sorted order
    __syncthreads();
    // X = Q Y (sorted columns) and the residual squares: thread per row, the
    // row of Q and of Z in registers, 8 output columns at a time
    for (int i = tid; i < n; i += blockDim.x) {
        double q[32], z[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) {
            q[m] = m < p ? Qs[i * pp + m] : 0.0;
            z[m] = m < p ? Zs[i * pp + m] : 0.0;
        }
        for (int j0 = 0; j0 < p; j0 += 8) {
            double x[8], zz[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = zz[u] = 0.0;
#pragma unroll
            for (int m = 0; m < 32; ++m) {
                if (m >= p) break;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double y = j0 + u < p ? Y[m * pp + j0 + u] : 0.0;
                    x[u] = fma(q[m], y, x[u]);
                    zz[u] = fma(z[m], y, zz[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int j = j0 + u;
                if (j >= p) break;
                X[static_cast<size_t>(i) * p + j] = x[u];
                const double rr = zz[u] - H[j * pp + j] * x[u];
                R2[j * n + i] = rr * rr;
            }
        }
    }
    __syncthreads();
    TK_T(6);
    for (int j = warp; j < p; j += nw) {  // a warp per column
        double s = 0.0;
        for (int i = lane; i < n; i += 32) s += R2[j * n + i];
        s = tk_warp_sum(s);
        if (lane == 0) {
            out[j] = H[j * pp + j];
            out[p + j] = sqrt(s);
        }
    }
    double tr = 0.0;
    for (int i = tid; i < n; i += blockDim.x) tr += G[static_cast<size_t>(i) * n + i];
    tr = tk_block_sum(tr, red);
    if (tid == 0) out[2 * p] = tr;
}

}  // namespace

#ifdef TCB_TOPK_TIMING
void topk_phase_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_tk_phase, sizeof(unsigned long long) * 16); }
#endif

bool topk_supported(u64 n, int p) {  // shared-memory footprints: tk_rr (3 n p + 2 p^2) and tk_gq (n (p + 8))
    return p >= 8 && p <= 32 && n >= static_cast<u64>(2 * p) && n <= 256;
}

void topk_eig(const double* G, u64 n64, int p, int extra_iters, double* X, std::vector<double>& theta,
              std::vector<double>& resid, double& trace, cudaStream_t s) {
    ProfScope prof_scope(kEig, s);
    const int n = static_cast<int>(n64);
    static bool attr = [] {
        cudaFuncSetAttribute(tk_gq, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(tk_cqr, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(tk_rr, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        return true;
    }();
    (void)attr;
    DevBuf<double> W(n64 * p, s), Z(n64 * p, s), out(2 * p + 2, s);
    TCB_CUDA(cudaMemsetAsync(out.p, 0, (2 * p + 2) * sizeof(double), s));
    int* fail = reinterpret_cast<int*>(out.p + 2 * p + 1);
    tk_random<<<cdiv(n64 * p, 256), 256, 0, s>>>(W.p, n, p);
    const size_t gsm = (8 * static_cast<size_t>(n) + static_cast<size_t>(n) * p) * sizeof(double);
    const size_t qsm = (static_cast<size_t>(n) + 64) * 33 * sizeof(double);
    const size_t rsm = (2 * static_cast<size_t>(n) * (p + 1) + 2 * static_cast<size_t>(p) * (p + 1) +
                        static_cast<size_t>(p) * n) * sizeof(double);
    for (int it = 0; it <= extra_iters; ++it) {
        tk_gq<<<cdiv(n64, 8), 256, gsm, s>>>(G, W.p, n, p, Z.p);
        tk_cqr<<<1, kTkQrThreads, qsm, s>>>(Z.p, n, p, W.p, fail);
    }
    tk_gq<<<cdiv(n64, 8), 256, gsm, s>>>(G, W.p, n, p, Z.p);
    tk_rr<<<1, kTkRrThreads, rsm, s>>>(G, W.p, Z.p, n, p, X, out.p);
    count_launch(2 * (extra_iters + 1) + 3);
    TCB_LAUNCH();
    std::vector<double> h(2 * p + 2);
    out.download(h.data(), 2 * p + 2);
    TCB_CUDA(cudaStreamSynchronize(s));
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
