// Device symmetric eigensolver for the per-mode Gram (n <= 1024, fp64):
// the SelfAdjointEigenSolver call of sthosvd.cpp:80-90, re-designed for B200.
//
//  1. Householder tridiagonalisation: one 8-CTA thread-block cluster, matrix in
//     L2, rows interleaved over the CTAs, two hardware cluster barriers/step.
//  2. All eigenvalues by Sturm-count bisection, one thread per eigenvalue.
//  3. Top-r eigenvectors of the tridiagonal by inverse iteration with
//     modified Gram-Schmidt inside eigenvalue clusters (LAPACK dstein scheme);
//     independent clusters run in parallel CTAs.
//  4. Back-transform U = Q Z (warp per column) and the column sign convention
//     of sthosvd.cpp:103-110.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cmath>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace tcb {

namespace {

constexpr int kCluster = 8;
constexpr int kTriThreads = 512;

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < nw; ++i) t += sh[i];
    return t;
}

// A: row-major n x n symmetric (overwritten).  Outputs d[n], e[n-1],
// V[k*n + i] (Householder vector of step k, entries i >= k+1), tau[k].
__global__ void __launch_bounds__(kTriThreads) tridiag_kernel(double* __restrict__ A, int n, double* __restrict__ d,
                                                             double* __restrict__ e, double* __restrict__ V,
                                                             double* __restrict__ tau, double* __restrict__ P) {
    cg::cluster_group cl = cg::this_cluster();
    const int rank = static_cast<int>(cl.block_rank());
    extern __shared__ double sh_tri[];
    double* v = sh_tri;          // n
    double* w = sh_tri + n;      // n
    double* red = sh_tri + 2 * n;  // 32
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;
        // x = A[k][k+1..n-1] (row k == column k by symmetry), redundantly in every CTA
        double ss = 0.0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const double x = __ldcg(A + static_cast<size_t>(k) * n + k + 1 + i);
            v[i] = x;
            ss += x * x;
        }
        const double alpha = sqrt(block_sum(ss, red));
        const double x0 = v[0];
        const double beta = x0 >= 0.0 ? -alpha : alpha;
        __syncthreads();
        if (threadIdx.x == 0) v[0] = x0 - beta;
        __syncthreads();
        double vv = 0.0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) vv += v[i] * v[i];
        vv = block_sum(vv, red);
        const double t = (alpha == 0.0 || vv == 0.0) ? 0.0 : 2.0 / vv;
        if (rank == 0) {
            if (threadIdx.x == 0) {
                e[k] = t == 0.0 ? x0 : beta;
                tau[k] = t;
                d[k] = __ldcg(A + static_cast<size_t>(k) * n + k);
            }
            for (int i = threadIdx.x; i < m; i += blockDim.x) V[static_cast<size_t>(k) * n + k + 1 + i] = v[i];
        }
        if (t != 0.0) {
            // p_i = t * sum_j A[i][j] v_j for owned rows i (warp per row)
            for (int r = k + 1 + rank + kCluster * warp; r < n; r += kCluster * nwarp) {
                const double* row = A + static_cast<size_t>(r) * n + k + 1;
                double s = 0.0;
                for (int j = lane; j < m; j += 32) s += __ldcg(row + j) * v[j];
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) P[r] = t * s;
            }
            cl.sync();
            double pv = 0.0;
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const double p = __ldcg(P + k + 1 + i);
                w[i] = p;
                pv += p * v[i];
            }
            const double K = 0.5 * t * block_sum(pv, red);
            for (int i = threadIdx.x; i < m; i += blockDim.x) w[i] -= K * v[i];
            __syncthreads();
            for (int r = k + 1 + rank + kCluster * warp; r < n; r += kCluster * nwarp) {
                double* row = A + static_cast<size_t>(r) * n + k + 1;
                const double vi = v[r - k - 1], wi = w[r - k - 1];
                for (int j = lane; j < m; j += 32) row[j] = __ldcg(row + j) - (vi * w[j] + wi * v[j]);
            }
        }
        cl.sync();
    }
    if (rank == 0 && threadIdx.x == 0) {
        if (n >= 2) {
            d[n - 2] = __ldcg(A + static_cast<size_t>(n - 2) * n + n - 2);
            e[n - 2] = __ldcg(A + static_cast<size_t>(n - 1) * n + n - 2);
        }
        d[n - 1] = __ldcg(A + static_cast<size_t>(n - 1) * n + n - 1);
    }
}

// Sturm count: number of eigenvalues of T strictly below x.
__device__ __forceinline__ int sturm(const double* d, const double* e2, int n, double x, double pivmin) {
    double q = d[0] - x;
    int c = q < 0.0;
    for (int i = 1; i < n; ++i) {
        if (fabs(q) < pivmin) q = -pivmin;
        q = (d[i] - x) - e2[i - 1] / q;
        c += q < 0.0;
    }
    return c;
}

// one thread per eigenvalue; ascending index j -> descending slot n-1-j
__global__ void bisect_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n,
                              double* __restrict__ evals_desc) {
    extern __shared__ double sh_bis[];
    double* d = sh_bis;
    double* e2 = sh_bis + n;
    double gl = DBL_MAX, gu = -DBL_MAX, emax2 = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        d[i] = dg[i];
        if (i + 1 < n) e2[i] = eg[i] * eg[i];
    }
    __syncthreads();
    // Gershgorin bounds (every thread computes the same, cheap for n <= 1024)
    for (int i = 0; i < n; ++i) {
        const double r = (i > 0 ? fabs(eg[i - 1]) : 0.0) + (i + 1 < n ? fabs(eg[i]) : 0.0);
        gl = fmin(gl, d[i] - r);
        gu = fmax(gu, d[i] + r);
        if (i + 1 < n) emax2 = fmax(emax2, e2[i]);
    }
    const double tnorm = fmax(fabs(gl), fabs(gu));
    const double pivmin = DBL_MIN * fmax(1.0, emax2);
    gl -= 2.0 * DBL_EPSILON * tnorm * n + 2.0 * pivmin;
    gu += 2.0 * DBL_EPSILON * tnorm * n + 2.0 * pivmin;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double lo = gl, hi = gu;  // invariant: count(lo) <= j < count(hi)
    for (int it = 0; it < 80; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        if (sturm(d, e2, n, mid, pivmin) > j) hi = mid;
        else lo = mid;
    }
    evals_desc[n - 1 - j] = 0.5 * (lo + hi);
}

__device__ __forceinline__ double hash_unit(unsigned a, unsigned b) {
    unsigned h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    h *= 0x297A2D39u;
    h ^= h >> 15;
    return (static_cast<double>(h) / 4294967295.0) * 2.0 - 1.0;
}

// Inverse iteration for one eigenvalue cluster per CTA.
// clusters[c] = first descending index of cluster c (clusters[nc] = r).
// Z: column-major n x r.
__global__ void invit_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n,
                             const double* __restrict__ evals_desc, const int* __restrict__ clusters, double tnorm,
                             double* __restrict__ Z) {
    extern __shared__ double sh_inv[];
    double* a = sh_inv;          // U diagonal
    double* b = a + n;           // first superdiagonal
    double* c = b + n;           // multipliers
    double* dd = c + n;          // second superdiagonal
    double* x = dd + n;          // iterate
    double* red = x + n;         // 32
    int* piv = reinterpret_cast<int*>(red + 32);
    const int j0 = clusters[blockIdx.x], j1 = clusters[blockIdx.x + 1];
    const double eps = DBL_EPSILON;
    const double tol = eps * tnorm + DBL_MIN;
    double prev = 0.0;
    for (int j = j0; j < j1; ++j) {
        double lam = evals_desc[j];
        if (j > j0) {
            const double pertol = 10.0 * eps * fabs(lam) + 2.0 * DBL_MIN;
            if (prev - lam < pertol) lam = prev - pertol;
        }
        prev = lam;
        if (threadIdx.x == 0) {
            // LU with partial pivoting of T - lam I (LAPACK dlagtf scheme)
            for (int i = 0; i < n; ++i) {
                a[i] = dg[i] - lam;
                b[i] = i + 1 < n ? eg[i] : 0.0;
                c[i] = i + 1 < n ? eg[i] : 0.0;
                dd[i] = 0.0;
            }
            for (int k = 0; k + 1 < n; ++k) {
                if (fabs(a[k]) >= fabs(c[k])) {
                    const double mult = a[k] == 0.0 ? 0.0 : c[k] / a[k];
                    c[k] = mult;
                    a[k + 1] -= mult * b[k];
                    piv[k] = 0;
                } else {
                    const double mult = a[k] / c[k];
                    a[k] = c[k];
                    const double tmp = a[k + 1];
                    a[k + 1] = b[k] - mult * tmp;
                    if (k + 2 < n) {
                        dd[k] = b[k + 1];
                        b[k + 1] = -mult * dd[k];
                    }
                    b[k] = tmp;
                    c[k] = mult;
                    piv[k] = 1;
                }
            }
            for (int i = 0; i < n; ++i)
                if (fabs(a[i]) < tol) a[i] = a[i] < 0.0 ? -tol : tol;
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = hash_unit(static_cast<unsigned>(j), i);
        __syncthreads();
        for (int it = 0; it < 4; ++it) {
            if (threadIdx.x == 0) {
                // apply L^{-1} (with the recorded interchanges), then U^{-1}
                for (int k = 0; k + 1 < n; ++k) {
                    if (piv[k]) {
                        const double t = x[k];
                        x[k] = x[k + 1];
                        x[k + 1] = t - c[k] * x[k];
                    } else {
                        x[k + 1] -= c[k] * x[k];
                    }
                }
                double scale = 1.0;
                for (int k = n - 1; k >= 0; --k) {
                    double t = x[k];
                    if (k + 1 < n) t -= b[k] * x[k + 1];
                    if (k + 2 < n) t -= dd[k] * x[k + 2];
                    t /= a[k];
                    x[k] = t;
                    if (fabs(t) > 1e150) {  // rescale the partial solution
                        for (int q = k; q < n; ++q) x[q] *= 1e-150;
                        scale *= 1e-150;
                    }
                }
                (void)scale;
            }
            __syncthreads();
            // normalise, then orthogonalise against earlier members of the cluster
            double s = 0.0;
            for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i] * x[i];
            double inv = 1.0 / sqrt(block_sum(s, red));
            for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] *= inv;
            __syncthreads();
            for (int q = j0; q < j; ++q) {
                const double* zq = Z + static_cast<size_t>(q) * n;
                double dt = 0.0;
                for (int i = threadIdx.x; i < n; i += blockDim.x) dt += zq[i] * x[i];
                dt = block_sum(dt, red);
                for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] -= dt * zq[i];
                __syncthreads();
            }
            s = 0.0;
            for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i] * x[i];
            inv = 1.0 / sqrt(block_sum(s, red));
            for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] *= inv;
            __syncthreads();
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x) Z[static_cast<size_t>(j) * n + i] = x[i];
        __syncthreads();
    }
}

// U (row-major n x r) = H_0 ... H_{n-3} Z; warp per column
__global__ void backtransform_kernel(const double* __restrict__ V, const double* __restrict__ tau, int n, int r,
                                     const double* __restrict__ Z, double* __restrict__ U) {
    const int lane = threadIdx.x & 31;
    const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (col >= r) return;
    double z[32];  // n <= 1024: 32 entries per lane (entry i = lane + 32 q)
#pragma unroll
    for (int q = 0; q < 32; ++q) {
        const int i = lane + 32 * q;
        z[q] = i < n ? Z[static_cast<size_t>(col) * n + i] : 0.0;
    }
    for (int k = n - 3; k >= 0; --k) {
        const double t = tau[k];
        if (t == 0.0) continue;
        const double* vk = V + static_cast<size_t>(k) * n;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const int i = lane + 32 * q;
            if (i > k && i < n) s += vk[i] * z[q];
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        s *= t;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const int i = lane + 32 * q;
            if (i > k && i < n) z[q] -= s * vk[i];
        }
    }
#pragma unroll
    for (int q = 0; q < 32; ++q) {
        const int i = lane + 32 * q;
        if (i < n) U[static_cast<size_t>(i) * r + col] = z[q];
    }
}

__global__ void sign_kernel(double* __restrict__ U, int n, int r) {
    const int lane = threadIdx.x & 31;
    const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (col >= r) return;
    double best = -1.0;
    int bi = 0;
    for (int i = lane; i < n; i += 32) {
        const double a = fabs(U[static_cast<size_t>(i) * r + col]);
        if (a > best) {
            best = a;
            bi = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    if (U[static_cast<size_t>(bi) * r + col] < 0.0)
        for (int i = lane; i < n; i += 32) U[static_cast<size_t>(i) * r + col] = -U[static_cast<size_t>(i) * r + col];
}

// U (row-major n x r): column j /= sigma_j, then modified Gram-Schmidt; a
// column that collapses is replaced by the first unit vector orthogonal to
// the others (orthonormal completion for zero singular values).
__global__ void scale_mgs_kernel(double* __restrict__ U, int n, int r, const double* __restrict__ sigma) {
    extern __shared__ double sh_mgs[];
    double* red = sh_mgs;
    for (int j = 0; j < r; ++j) {
        const double sg = sigma[j];
        if (sg > 0.0)
            for (int i = threadIdx.x; i < n; i += blockDim.x) U[static_cast<size_t>(i) * r + j] /= sg;
        __syncthreads();
        for (int attempt = 0; attempt <= n; ++attempt) {
            if (attempt > 0)
                for (int i = threadIdx.x; i < n; i += blockDim.x)
                    U[static_cast<size_t>(i) * r + j] = (i == attempt - 1) ? 1.0 : 0.0;
            __syncthreads();
            double nrm0 = 0.0;
            for (int i = threadIdx.x; i < n; i += blockDim.x) nrm0 += U[static_cast<size_t>(i) * r + j] * U[static_cast<size_t>(i) * r + j];
            nrm0 = sqrt(block_sum(nrm0, red));
            for (int pass = 0; pass < 2; ++pass)
                for (int q = 0; q < j; ++q) {
                    double dt = 0.0;
                    for (int i = threadIdx.x; i < n; i += blockDim.x)
                        dt += U[static_cast<size_t>(i) * r + q] * U[static_cast<size_t>(i) * r + j];
                    dt = block_sum(dt, red);
                    for (int i = threadIdx.x; i < n; i += blockDim.x)
                        U[static_cast<size_t>(i) * r + j] -= dt * U[static_cast<size_t>(i) * r + q];
                    __syncthreads();
                }
            double nrm = 0.0;
            for (int i = threadIdx.x; i < n; i += blockDim.x) nrm += U[static_cast<size_t>(i) * r + j] * U[static_cast<size_t>(i) * r + j];
            nrm = sqrt(block_sum(nrm, red));
            if (nrm > 0.5 * nrm0 && nrm > 0.0) {
                for (int i = threadIdx.x; i < n; i += blockDim.x) U[static_cast<size_t>(i) * r + j] /= nrm;
                __syncthreads();
                break;
            }
            __syncthreads();
        }
    }
}

}  // namespace

std::vector<double> eig_values(const double* A, u64 n64, EigWork& w, cudaStream_t s) {
    ProfScope prof_scope(kEig, s);
    const int n = static_cast<int>(n64);
    if (n64 > 1024) throw Error("sthosvd: device eigensolver supports mode sizes up to 1024");
    w.n = n64;
    w.a = DevBuf<double>(n64 * n64, s);
    w.d = DevBuf<double>(n64, s);
    w.e = DevBuf<double>(n64 + 1, s);
    w.tau = DevBuf<double>(n64 + 1, s);
    w.evals = DevBuf<double>(n64, s);
    DevBuf<double> V(n64 * n64, s), P(n64, s);
    w.z = std::move(V);
    TCB_CUDA(cudaMemcpyAsync(w.a.p, A, n64 * n64 * sizeof(double), cudaMemcpyDeviceToDevice, s));
    w.tau.zero();
    if (n == 1) {
        TCB_CUDA(cudaMemcpyAsync(w.d.p, A, sizeof(double), cudaMemcpyDeviceToDevice, s));
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kCluster);
        cfg.blockDim = dim3(kTriThreads);
        cfg.dynamicSmemBytes = (2 * n + 32) * sizeof(double);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = kCluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        TCB_CUDA(cudaLaunchKernelEx(&cfg, tridiag_kernel, w.a.p, n, w.d.p, w.e.p, w.z.p, w.tau.p, P.p));
        count_launch();
    }
    const int bthreads = 128;
    bisect_kernel<<<cdiv(n64, bthreads), bthreads, 2 * n * sizeof(double), s>>>(w.d.p, w.e.p, n, w.evals.p);
    count_launch();
    TCB_LAUNCH();
    std::vector<double> ev(n64);
    w.evals.download(ev.data(), n64);
    TCB_CUDA(cudaStreamSynchronize(s));
    return ev;
}

void eig_vectors(EigWork& w, u64 r64, double* U, cudaStream_t s) {
    ProfScope prof_scope(kEig, s);
    const int n = static_cast<int>(w.n), r = static_cast<int>(r64);
    std::vector<double> ev(w.n), d(w.n), e(w.n + 1);
    w.evals.download(ev.data(), w.n);
    w.d.download(d.data(), w.n);
    w.e.download(e.data(), w.n > 1 ? w.n - 1 : 0);
    TCB_CUDA(cudaStreamSynchronize(s));
    double tnorm = 0.0;
    for (int i = 0; i < n; ++i) {
        const double rr = std::fabs(d[i]) + (i > 0 ? std::fabs(e[i - 1]) : 0.0) + (i + 1 < n ? std::fabs(e[i]) : 0.0);
        tnorm = std::max(tnorm, rr);
    }
    if (!(tnorm > 0.0)) tnorm = 1.0;  // zero matrix: any orthonormal basis is an eigenbasis
    const double ortol = 1e-3 * tnorm;
    std::vector<int> cl{0};
    for (int j = 1; j < r; ++j)
        if (ev[j - 1] - ev[j] > ortol) cl.push_back(j);
    cl.push_back(r);
    DevBuf<int> clb(cl.size(), s);
    clb.upload(cl.data(), cl.size());
    DevBuf<double> Z(static_cast<u64>(n) * r, s);
    const size_t smem = (5 * n + 32) * sizeof(double) + n * sizeof(int);
    invit_kernel<<<static_cast<unsigned>(cl.size() - 1), 256, smem, s>>>(w.d.p, w.e.p, n, w.evals.p, clb.p, tnorm,
                                                                         Z.p);
    backtransform_kernel<<<cdiv(r64, 4), 128, 0, s>>>(w.z.p, w.tau.p, n, r, Z.p, U);
    count_launch(2);
    TCB_LAUNCH();
}

void fix_column_signs(double* U, u64 n, u64 r, cudaStream_t s) {
    ProfScope prof_scope(kEig, s);
    sign_kernel<<<cdiv(r, 4), 128, 0, s>>>(U, static_cast<int>(n), static_cast<int>(r));
    count_launch();
    TCB_LAUNCH();
}

void scale_orthonormalize(double* U, u64 n, u64 r, const double* sigma, cudaStream_t s) {
    ProfScope prof_scope(kEig, s);
    scale_mgs_kernel<<<1, 256, 32 * sizeof(double), s>>>(U, static_cast<int>(n), static_cast<int>(r), sigma);
    count_launch();
    TCB_LAUNCH();
}

}  // namespace tcb
