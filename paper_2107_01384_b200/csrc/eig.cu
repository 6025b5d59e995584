// Device symmetric eigensolver for the per-mode Gram (n <= 1024, fp64):
// the SelfAdjointEigenSolver call of sthosvd.cpp:80-90, re-designed for B200.
//
//  1. Householder tridiagonalisation on one 8-CTA thread-block cluster.
//     n <= 448: the matrix lives in distributed shared memory (rows
//     interleaved over the CTAs); p-slices and the next column are pushed to
//     every CTA with DSMEM stores, two hardware cluster barriers per step.
//     Larger n: same schedule with the matrix in L2.
//  2. All eigenvalues by Sturm-count multisection: one warp per eigenvalue,
//     32 probes per round (5 bits/round), reciprocal via rcp.approx + Newton.
//  3. Top-r eigenvectors of the tridiagonal by inverse iteration, one CTA
//     per vector (all in parallel), then modified Gram-Schmidt inside tight
//     eigenvalue clusters (gap <= 1e-6 ||T||), independent clusters in parallel.
//  4. Back-transform U = Q Z with reflector chunks staged in shared memory,
//     and the column sign convention of sthosvd.cpp:103-110.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace tcb {

namespace {

constexpr int kCluster = 8;
constexpr int kTriThreads = 512;
constexpr int kDsmemMaxN = 600;  // nloc <= 38: at most 2 row slots per warp

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

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------- tridiagonalisation (DSMEM)
// Row i lives in CTA (i % C), local slot i / C (C = 16-CTA cluster, the
// non-portable maximum).  One warp per row slot (slot li -> warp li % nw,
// nw = min(nloc, 32) warps, so up to 1024 threads hide shared-memory
// latency); lanes stride the columns.  Per step k:
//   A. every CTA derives alpha/beta/tau from the replicated column k (rowk),
//      whose |x|^2 partials were accumulated while it was built;
//   B. each warp forms p_i = tau A_i . v for its active rows (xor butterfly:
//      every lane ends with the same bits) and lanes 0..C-1 push
//      {p_i, pre-update A_i,k+1} to CTA `lane` with one 16-byte st.async that
//      completes transaction bytes on the receiver's mbarrier; the CTA's sum
//      of p_i v_i (fixed order) is pushed to every CTA the same way;
//   -- wait on the local mbarrier for 16 m + 8 C bytes (no cluster barrier,
//      no GPU-scope fence) --
//   C. K = tau/2 (sum of the C partials, same order on every CTA); each warp
//      updates its rows, A_ij -= v_i w_j + w_i v_j with w = p - K v, and every
//      CTA rebuilds the updated row k+1 (the next column) from the pushed
//      pre-update column with one shared expression; one CTA barrier.
// Step k+1's pushes into a CTA's buffer (k+1)&1 are issued only after the
// sender passed step k's wait, i.e. after every CTA finished step k-1, the
// last reader of that buffer, so double buffering is enough.
// Outputs d, e, V (reflector k at V[k*n + i], i >= k+1), tau.
constexpr int kTdCluster = 16;
constexpr int kTdMaxWarps = 32;
constexpr int kTdMaxRowsPerWarp = 2;  // nloc <= 64, i.e. n <= 1024

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned cluster_map(unsigned addr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_f64(unsigned raddr, double v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v2f64(unsigned raddr, double a, double b, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(unsigned bar, unsigned tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

#ifdef TCB_TRIDIAG_TIMING
__device__ unsigned long long g_tri_phase[16 * 10];
#define TRI_T(i)                                           \
    do {                                                   \
        const long long now_ = clock64();                  \
        if (threadIdx.x == 0) tacc[i] += now_ - tprev;     \
        tprev = now_;                                      \
    } while (0)
#else
#define TRI_T(i) \
    do {         \
    } while (0)
#endif
__global__ void __launch_bounds__(1024) tridiag_dsmem(const double* __restrict__ Ag, int n, double* __restrict__ d,
                                                      double* __restrict__ e, double* __restrict__ V,
                                                      double* __restrict__ tau) {
    constexpr int C = kTdCluster;
#ifdef TCB_TRIDIAG_TIMING
    long long tacc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tprev = clock64();
#endif
    cg::cluster_group cl = cg::this_cluster();
    const int rank = static_cast<int>(cl.block_rank());
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) unsigned long long mbar[2];
    __shared__ double red[kTdMaxWarps];        // per-warp sums of p_i v_i
    __shared__ double ssbuf[2 * kTdMaxWarps];  // per-warp |next column|^2 partials
    __shared__ double kbuf[2 * C];             // remote-written CTA sums of p_i v_i
    const int nloc = (n + C - 1) / C;
    const int nw = static_cast<int>(blockDim.x >> 5);
    double* A = sm;                                                           // nloc x n
    double2* pobuf = reinterpret_cast<double2*>(A + ((nloc * n + 1) & ~1));  // 2 x n {p_i, pre-update A_i,k+1}
    double* rbuf = reinterpret_cast<double*>(pobuf + 2 * n);                  // 2 x n replicated column k
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(smem_addr(&mbar[0]), 1);
        mbar_init(smem_addr(&mbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int li = 0; li < nloc; ++li) {
        const int gi = li * C + rank;
        for (int j = threadIdx.x; j < n; j += blockDim.x)
            A[li * n + j] = gi < n ? Ag[static_cast<size_t>(gi) * n + j] : 0.0;
    }
    {
        double ss = 0.0;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            const double x = Ag[j];
            rbuf[j] = x;
            if (j >= 1) ss += x * x;
        }
        ss = warp_sum(ss);
        if (lane == 0) ssbuf[warp] = ss;
    }
    __syncthreads();
    cl.sync();
    // push target of this lane: CTA lane % C (loop invariant)
    const unsigned dst = static_cast<unsigned>(lane & (C - 1));
    const unsigned rpo = cluster_map(smem_addr(pobuf), dst), rkb = cluster_map(smem_addr(kbuf), dst);
    const unsigned rbar[2] = {cluster_map(smem_addr(&mbar[0]), dst), cluster_map(smem_addr(&mbar[1]), dst)};
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;
        const int buf = k & 1;
        const double* rowk = rbuf + buf * n;
        double* rnext = rbuf + (buf ^ 1) * n;
        const double2* po = pobuf + buf * n;
        const double* kb = kbuf + buf * C;
        TRI_T(0);
        if (threadIdx.x == 0) mbar_arrive_expect(smem_addr(&mbar[buf]), static_cast<unsigned>(16 * m + 8 * C));
        // this warp's active row slots (warp-uniform)
        int li[kTdMaxRowsPerWarp];
        bool act[kTdMaxRowsPerWarp];
#pragma unroll
        for (int r = 0; r < kTdMaxRowsPerWarp; ++r) {
            li[r] = warp + r * nw;
            const int gi = li[r] * C + rank;
            act[r] = li[r] < nloc && gi >= k + 1 && gi < n;
        }
        // B1. matvec over columns j >= k+2 (independent of alpha, so it overlaps the sqrt/divide)
        double acc[kTdMaxRowsPerWarp];
#pragma unroll
        for (int r = 0; r < kTdMaxRowsPerWarp; ++r) {
            acc[r] = 0.0;
            if (act[r]) {
                const double* Ar = A + li[r] * n;
                double a2 = 0.0;
                int j = k + 2 + lane;
                for (; j + 32 < n; j += 64) {
                    acc[r] = fma(Ar[j], rowk[j], acc[r]);
                    a2 = fma(Ar[j + 32], rowk[j + 32], a2);
                }
                if (j < n) acc[r] = fma(Ar[j], rowk[j], acc[r]);
                acc[r] += a2;
            }
        }
        // A. reflector of column k
        double ss = 0.0;
        for (int q = 0; q < nw; ++q) ss += ssbuf[buf * kTdMaxWarps + q];
        const double alpha = sqrt(ss);
        const double x0 = rowk[k + 1];
        const double beta = x0 >= 0.0 ? -alpha : alpha;
        const double v0 = x0 - beta;
        const double vv = 2.0 * alpha * (alpha + fabs(x0));  // |x - beta e1|^2
        const double t = (alpha == 0.0 || vv == 0.0) ? 0.0 : 2.0 / vv;
        TRI_T(1);
        // B2. finish p_i, push {p_i, A_i,k+1} and the CTA's p.v partial
        double p[kTdMaxRowsPerWarp], vi[kTdMaxRowsPerWarp];
        double kp = 0.0;
#pragma unroll
        for (int r = 0; r < kTdMaxRowsPerWarp; ++r) {
            p[r] = 0.0;
            vi[r] = 0.0;
            if (act[r]) {
                const int gi = li[r] * C + rank;
                const double ak1 = A[li[r] * n + k + 1];
                double s = acc[r] + (lane == 0 ? ak1 * v0 : 0.0);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                p[r] = t * s;
                vi[r] = gi == k + 1 ? v0 : rowk[gi];
                kp += p[r] * vi[r];
                if (lane < C)
                    st_async_v2f64(rpo + static_cast<unsigned>((buf * n + gi) * sizeof(double2)), p[r], ak1,
                                   rbar[buf]);
            }
        }
        if (lane == 0) red[warp] = kp;
        TRI_T(9);
        __syncthreads();
        TRI_T(2);
        if (warp == 0 && lane < C) {
            double s = 0.0;
            for (int q = 0; q < nw; ++q) s += red[q];
            st_async_f64(rkb + static_cast<unsigned>((buf * C + rank) * sizeof(double)), s, rbar[buf]);
        }
        TRI_T(3);
        mbar_wait(smem_addr(&mbar[buf]), static_cast<unsigned>((k >> 1) & 1));
        TRI_T(4);
        if (rank == k % C) {  // global outputs, off the exchange's critical path
            if (threadIdx.x == 0) {
                e[k] = t == 0.0 ? x0 : beta;
                tau[k] = t;
                d[k] = rowk[k];
            }
            for (int i = threadIdx.x; i < m; i += blockDim.x)
                V[static_cast<size_t>(k) * n + k + 1 + i] = i == 0 ? v0 : rowk[k + 1 + i];
        }
        // K = tau/2 p.v: butterfly over the C partials, identical bits on every lane and CTA
        double K = kb[lane & (C - 1)];
#pragma unroll
        for (int o = C / 2; o > 0; o >>= 1) K += __shfl_xor_sync(0xffffffffu, K, o);
        K *= 0.5 * t;
        const double wk1 = po[k + 1].x - K * v0;
        TRI_T(5);
        // C. rank-2 update of this warp's rows
#pragma unroll
        for (int r = 0; r < kTdMaxRowsPerWarp; ++r) {
            if (act[r]) {
                double* Ar = A + li[r] * n;
                const double wi = p[r] - K * vi[r];
                for (int j = k + 1 + lane; j < n; j += 32) {
                    const double vjj = j == k + 1 ? v0 : rowk[j], wj = po[j].x - K * vjj;
                    Ar[j] = Ar[j] - (vi[r] * wj + wi * vjj);
                }
            }
        }
        TRI_T(6);
        // updated row k+1 (= next column), rebuilt on every CTA from the pushed pre-update column
        double ssn = 0.0;
        for (int j = k + 1 + threadIdx.x; j < n; j += blockDim.x) {
            const double2 pj = po[j];
            const double vjj = j == k + 1 ? v0 : rowk[j], wj = pj.x - K * vjj;
            const double val = pj.y - (v0 * wj + wk1 * vjj);
            rnext[j] = val;
            if (j >= k + 2) ssn += val * val;
        }
        ssn = warp_sum(ssn);
        if (lane == 0) ssbuf[(buf ^ 1) * kTdMaxWarps + warp] = ssn;
        TRI_T(7);
        __syncthreads();
        TRI_T(8);
    }
#ifdef TCB_TRIDIAG_TIMING
    if (threadIdx.x == 0)
        for (int i = 0; i < 10; ++i) g_tri_phase[rank * 10 + i] = tacc[i];
#endif
    const double* rowl = rbuf + ((n - 2) & 1) * n;  // row n-2 after the last step
    if (rank == 0 && threadIdx.x == 0 && n >= 2) {
        d[n - 2] = rowl[n - 2];
        e[n - 2] = rowl[n - 1];
    }
    if (n >= 2 && (n - 1) % C == rank && threadIdx.x == 0) d[n - 1] = A[((n - 1) / C) * n + n - 1];
    cl.sync();  // no CTA leaves while cluster peers may still address its shared memory
}

// Same schedule with the matrix in L2 (n > kDsmemMaxN).
__global__ void __launch_bounds__(kTriThreads) tridiag_global(double* __restrict__ A, int n, double* __restrict__ d,
                                                             double* __restrict__ e, double* __restrict__ V,
                                                             double* __restrict__ tau, double* __restrict__ P) {
    cg::cluster_group cl = cg::this_cluster();
    const int rank = static_cast<int>(cl.block_rank());
    extern __shared__ double sh_tri[];
    double* v = sh_tri;
    double* w = sh_tri + n;
    double* red = sh_tri + 2 * n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;
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
            for (int r = k + 1 + rank + kCluster * warp; r < n; r += kCluster * nwarp) {
                const double* row = A + static_cast<size_t>(r) * n + k + 1;
                double s = 0.0;
                for (int j = lane; j < m; j += 32) s += __ldcg(row + j) * v[j];
                s = warp_sum(s);
                if (lane == 0) P[r] = t * s;
            }
            cl.sync();
            double pv = 0.0;
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const double q = __ldcg(P + k + 1 + i);
                w[i] = q;
                pv += q * v[i];
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

// ---------------------------------------------------------------- tridiagonalisation (whole GPU)
// Large n: one persistent CTA per SM (cooperative launch), the matrix in L2.
// Row r belongs to CTA r % G (warp (r / G) % nw).  Step k:
//   1. wait for row k (the pivot row, updated eagerly by its owner at step
//      k-1 and published with a release flag), read it; every CTA derives
//      alpha / beta / tau / v redundantly (identical arithmetic, identical
//      values everywhere);
//   2. every owned row r > k takes the previous step's deferred rank-2 update
//      (A_rj -= v_r w_j + w_r v_j) and, in the same pass, its dot product
//      p_r = tau A_r . v: one read and one write of the trailing matrix per step;
//   3. grid barrier (all of p), then every CTA forms K = tau/2 p.v and
//      w = p - K v in the same fixed order;
//   4. the owner of row k+1 applies this step's update to it at once (the next
//      pivot row) and raises its flag; the other rows keep it deferred.
// Same reflector convention and outputs as the cluster kernels.
constexpr int kCoopThreads = 512;

__device__ __forceinline__ void coop_barrier(unsigned* ctr, unsigned& phase) {
    __syncthreads();
    if (threadIdx.x == 0) {
        ++phase;
        __threadfence();
        atomicAdd(ctr, 1u);
        const unsigned target = phase * gridDim.x;
        while (*reinterpret_cast<volatile unsigned*>(ctr) < target) {
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kCoopThreads, 1) tridiag_coop(double* __restrict__ A, int n, double* __restrict__ d,
                                                               double* __restrict__ e, double* __restrict__ V,
                                                               double* __restrict__ tau, double* __restrict__ P,
                                                               unsigned* __restrict__ ctr, int* __restrict__ flags) {
    extern __shared__ double sh_coop[];
    double* v = sh_coop;
    double* w = v + n;
    double* vp = w + n;
    double* wp = vp + n;
    double* red = wp + n;
    const int G = static_cast<int>(gridDim.x), cta = static_cast<int>(blockIdx.x);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned phase = 0;
    bool pend = false;  // a deferred update (vp, wp) of the previous step
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;
        if (k > 0) {
            if (threadIdx.x == 0) {
                while (*reinterpret_cast<volatile int*>(flags + k) == 0) {
                }
                __threadfence();
            }
            __syncthreads();
        }
        // one reduction: the tail |x_1..|^2 gives both alpha and |v|^2
        double ss = 0.0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const double x = __ldcg(A + static_cast<size_t>(k) * n + k + 1 + i);
            v[i] = x;
            if (i > 0) ss += x * x;
        }
        const double tail = block_sum(ss, red);
        const double x0 = v[0];
        const double alpha = sqrt(x0 * x0 + tail);
        const double beta = x0 >= 0.0 ? -alpha : alpha;
        const double v0 = x0 - beta;
        const double vv = v0 * v0 + tail;
        __syncthreads();
        if (threadIdx.x == 0) v[0] = v0;
        __syncthreads();
        const double t = (alpha == 0.0 || vv == 0.0) ? 0.0 : 2.0 / vv;
        if (cta == 0) {
            if (threadIdx.x == 0) {
                e[k] = t == 0.0 ? x0 : beta;
                tau[k] = t;
                d[k] = __ldcg(A + static_cast<size_t>(k) * n + k);
            }
            for (int i = threadIdx.x; i < m; i += blockDim.x) V[static_cast<size_t>(k) * n + k + 1 + i] = v[i];
        }
        // owned rows r > k: deferred update of step k-1 (columns > k) + p_r
        for (int q = warp;; q += nw) {
            const int r = cta + G * q;
            if (r >= n) break;
            if (r <= k) continue;
            double* __restrict__ row = A + static_cast<size_t>(r) * n + k + 1;
            double s = 0.0;
            if (pend) {
                const double vr = vp[r - k], wr = wp[r - k];
                // 4 columns per lane in flight: every load is issued before the stores
                for (int j0 = lane; j0 < m; j0 += 128) {
                    double a[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) a[u] = j0 + 32 * u < m ? __ldcg(row + j0 + 32 * u) : 0.0;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int j = j0 + 32 * u;
                        if (j < m) {
                            a[u] -= vr * wp[j + 1] + wr * vp[j + 1];
                            row[j] = a[u];
                            s += a[u] * v[j];
                        }
                    }
                }
            } else {
                for (int j = lane; j < m; j += 32) s += __ldcg(row + j) * v[j];
            }
            s = warp_sum(s);
            if (lane == 0) P[r] = t * s;
        }
        coop_barrier(ctr, phase);
        double pv = 0.0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const double q = __ldcg(P + k + 1 + i);
            w[i] = q;
            pv += q * v[i];
        }
        const double K = 0.5 * t * block_sum(pv, red);
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            w[i] -= K * v[i];
            vp[i] = v[i];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += blockDim.x) wp[i] = w[i];
        __syncthreads();
        // vp / wp now index rows k+1+i: shift by one so that vp[r - (k+1)] ... the
        // next step reads vp[r - (k + 1)] as vp[r - k'] with k' = k + 1
        pend = t != 0.0;
        if ((k + 1) % G == cta && warp == 0) {  // the next pivot row, at once
            double* row = A + static_cast<size_t>(k + 1) * n + k + 1;
            if (pend) {
                const double v0 = v[0], w0 = w[0];
                for (int j = lane; j < m; j += 32) row[j] = __ldcg(row + j) - (v0 * w[j] + w0 * v[j]);
            }
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicExch(flags + k + 1, 1);
        }
        __syncthreads();
    }
    // the last two rows: row n-2 is current (pivot update), row n-1 takes its deferred update
    coop_barrier(ctr, phase);
    if (n >= 2 && cta == (n - 1) % G && threadIdx.x == 0) {
        const int k = n - 2;  // vp/wp belong to step k-1 = n-3; row n-1 <-> index 1
        double a_nn = __ldcg(A + static_cast<size_t>(n - 1) * n + n - 1);
        double a_n1 = __ldcg(A + static_cast<size_t>(n - 1) * n + n - 2);
        if (pend && n >= 3) {
            const double vr = vp[(n - 1) - k], wr = wp[(n - 1) - k];
            a_nn -= vr * wp[(n - 1) - k] + wr * vp[(n - 1) - k];
            a_n1 -= vr * wp[(n - 2) - k] + wr * vp[(n - 2) - k];
        }
        d[n - 2] = __ldcg(A + static_cast<size_t>(n - 2) * n + n - 2);
        e[n - 2] = a_n1;
        d[n - 1] = a_nn;
    }
}

// The same algorithm with every CTA's rows resident in shared memory (Q rows of
// n doubles per CTA: n <= ~1700 on 148 SMs): the per-step update + dot product
// of a row is a pass over shared memory instead of an L2 round trip per 128
// columns, so a step costs the pivot chain and one grid barrier.  The pivot
// row is still published through global memory (with its flag); P through
// global memory as before.  Row q of CTA c is matrix row c + G q; the warps
// split each row into S column segments (Q S <= warps).
__global__ void __launch_bounds__(kCoopThreads, 1) tridiag_coop_smem(double* __restrict__ A, int n,
                                                                    double* __restrict__ d, double* __restrict__ e,
                                                                    double* __restrict__ V, double* __restrict__ tau,
                                                                    double* __restrict__ P, unsigned* __restrict__ ctr,
                                                                    int* __restrict__ flags, int Q, int S) {
    extern __shared__ double sh_coop[];
    double* rows = sh_coop;
    double* v = rows + static_cast<size_t>(Q) * n;
    double* w = v + n;
    double* vp = w + n;
    double* wp = vp + n;
    double* red = wp + n;
    double* part = red + 32;
    const int G = static_cast<int>(gridDim.x), cta = static_cast<int>(blockIdx.x);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int q = 0; q < Q; ++q) {
        const int r = cta + G * q;
        if (r >= n) break;
        for (int j = threadIdx.x; j < n; j += blockDim.x) rows[static_cast<size_t>(q) * n + j] = A[static_cast<size_t>(r) * n + j];
    }
    __syncthreads();
    unsigned phase = 0;
    bool pend = false;
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;
        if (k > 0) {
            if (threadIdx.x == 0) {
                while (*reinterpret_cast<volatile int*>(flags + k) == 0) {
                }
                __threadfence();
            }
            __syncthreads();
        }
        double ss = 0.0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const double x = __ldcg(A + static_cast<size_t>(k) * n + k + 1 + i);
            v[i] = x;
            if (i > 0) ss += x * x;
        }
        const double tail = block_sum(ss, red);
        const double x0 = v[0];
        const double alpha = sqrt(x0 * x0 + tail);
        const double beta = x0 >= 0.0 ? -alpha : alpha;
        const double v0 = x0 - beta;
        const double vv = v0 * v0 + tail;
        __syncthreads();
        if (threadIdx.x == 0) v[0] = v0;
        __syncthreads();
        const double t = (alpha == 0.0 || vv == 0.0) ? 0.0 : 2.0 / vv;
        if (cta == 0) {
            if (threadIdx.x == 0) {
                e[k] = t == 0.0 ? x0 : beta;
                tau[k] = t;
                d[k] = __ldcg(A + static_cast<size_t>(k) * n + k);
            }
            for (int i = threadIdx.x; i < m; i += blockDim.x) V[static_cast<size_t>(k) * n + k + 1 + i] = v[i];
        }
        // (row, segment) items: deferred update of step k-1 + partial dot with v
        const int seg_len = ((m + S - 1) / S + 31) & ~31;
        for (int it = warp; it < Q * S; it += nw) {
            const int q = it / S, sg = it - q * S;
            const int r = cta + G * q;
            double s = 0.0;
            if (r > k && r < n) {
                double* __restrict__ row = rows + static_cast<size_t>(q) * n + k + 1;
                const int j1 = min(m, (sg + 1) * seg_len);
                if (pend) {
                    const double vr = vp[r - k], wr = wp[r - k];
                    for (int j = sg * seg_len + lane; j < j1; j += 32) {
                        const double a = row[j] - (vr * wp[j + 1] + wr * vp[j + 1]);
                        row[j] = a;
                        s += a * v[j];
                    }
                } else {
                    for (int j = sg * seg_len + lane; j < j1; j += 32) s += row[j] * v[j];
                }
            }
            s = warp_sum(s);
            if (lane == 0) part[it] = s;
        }
        __syncthreads();
        if (threadIdx.x < Q) {
            const int r = cta + G * static_cast<int>(threadIdx.x);
            if (r > k && r < n) {
                double s = 0.0;
                for (int sg = 0; sg < S; ++sg) s += part[threadIdx.x * S + sg];
                P[r] = t * s;
            }
        }
        coop_barrier(ctr, phase);
        double pv = 0.0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const double q = __ldcg(P + k + 1 + i);
            w[i] = q;
            pv += q * v[i];
        }
        const double K = 0.5 * t * block_sum(pv, red);
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            w[i] -= K * v[i];
            vp[i] = v[i];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += blockDim.x) wp[i] = w[i];
        __syncthreads();
        pend = t != 0.0;
        if ((k + 1) % G == cta && warp == 0) {  // the next pivot row: update, publish, flag
            double* row = rows + static_cast<size_t>((k + 1) / G) * n + k + 1;
            double* out = A + static_cast<size_t>(k + 1) * n + k + 1;
            const double v0 = v[0], w0 = w[0];
            for (int j = lane; j < m; j += 32) {
                const double a = pend ? row[j] - (v0 * w[j] + w0 * v[j]) : row[j];
                row[j] = a;
                out[j] = a;
            }
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicExch(flags + k + 1, 1);
        }
        __syncthreads();
    }
    coop_barrier(ctr, phase);
    if (n >= 2 && cta == (n - 1) % G && threadIdx.x == 0) {
        const int k = n - 2;
        const double* rl = rows + static_cast<size_t>((n - 1) / G) * n;
        double a_nn = rl[n - 1];
        double a_n1 = rl[n - 2];
        if (pend && n >= 3) {
            const double vr = vp[(n - 1) - k], wr = wp[(n - 1) - k];
            a_nn -= vr * wp[(n - 1) - k] + wr * vp[(n - 1) - k];
            a_n1 -= vr * wp[(n - 2) - k] + wr * vp[(n - 2) - k];
        }
        d[n - 2] = __ldcg(A + static_cast<size_t>(n - 2) * n + n - 2);
        e[n - 2] = a_n1;
        d[n - 1] = a_nn;
    }
}

// ---------------------------------------------------------------- eigenvalues
__device__ __forceinline__ double frcp(double q) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
    y = fma(y, fma(-q, y, 1.0), y);
    y = fma(y, fma(-q, y, 1.0), y);
    return y;
}

// Sturm counts (eigenvalues of T below x) for PR probes at once: independent
// division chains per thread hide the fp64 latency.
// Sturm count (eigenvalues < x) by the three-term recurrence
// p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2} = det(T_i - x I) on a T scaled by a
// power of two to ||T|| < 1.  The critical chain is one FMA per step (the
// e^2 p_{i-2} product is ready a step early); a count is a sign change of
// consecutive terms (XOR of sign bits, off the chain).  e^2 == 0 needs no
// restart: the sequence continues as a product and the changes add up per
// block.  Every 8 steps both terms are rescaled by an exact power of two.
// Each step's rounding is a relative perturbation of d_i - x and e^2, so the
// count is exact for a matrix within a few ulps of ||T||, as for the ratio
// form.  An exact zero term (measure zero) sets `hit` and the caller recounts
// with the ratio form's q -> -pivmin rule.
__device__ __forceinline__ int dexp(double v) {
    return static_cast<int>((__double_as_longlong(v) >> 52) & 0x7FF) - 1023;
}
__device__ __forceinline__ unsigned sgn(double v) {
    return static_cast<unsigned>(__double_as_longlong(v) >> 63) & 1u;
}
template <int PR>
__device__ __forceinline__ void sturm_poly(const double* ds, const double* e2s, int n, const double (&x)[PR],
                                           int (&c)[PR], bool& hit) {
    double p0[PR], p1[PR];
    unsigned zero = 0;
#pragma unroll
    for (int u = 0; u < PR; ++u) {
        p0[u] = 1.0;
        p1[u] = ds[0] - x[u];
        c[u] = static_cast<int>(sgn(p1[u]));
        zero |= p1[u] == 0.0;
    }
    auto step = [&](int i) {
        const double di = ds[i], ei = e2s[i - 1];
#pragma unroll
        for (int u = 0; u < PR; ++u) {
            const double t = ei * p0[u];
            const double p = fma(di - x[u], p1[u], -t);
            c[u] += static_cast<int>(sgn(p) ^ sgn(p1[u]));
            zero |= p == 0.0;
            p0[u] = p1[u];
            p1[u] = p;
        }
    };
    int i = 1;
    for (; i + 8 <= n; i += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) step(i + k);
#pragma unroll
        for (int u = 0; u < PR; ++u) {
            const int ex = max(dexp(p0[u]), dexp(p1[u]));
            const double sc = __longlong_as_double(static_cast<long long>(1023 - ex) << 52);
            p0[u] *= sc;
            p1[u] *= sc;
        }
    }
    for (; i < n; ++i) step(i);
    hit = zero != 0;
}
// reference count for the rare exact-zero probes: LAPACK's ratio recurrence
__device__ __noinline__ int sturm_ratio(const double* ds, const double* e2s, int n, double x, double pivmin) {
    double q = ds[0] - x;
    int c = q < 0.0;
    for (int i = 1; i < n; ++i) {
        if (fabs(q) < pivmin) q = -pivmin;
        q = (ds[i] - x) - e2s[i - 1] / q;
        c += q < 0.0;
    }
    return c;
}

// one warp per eigenvalue (ascending index j), 64 probes per round (6 bits)
constexpr int kProbes = 2;
__global__ void multisect_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n,
                                 double* __restrict__ evals_desc) {
    extern __shared__ double sh_bis[];
    double* d = sh_bis;
    double* e2 = sh_bis + n;
    __shared__ double bounds[4];
    __shared__ double red3[3][32];
    {  // Gershgorin interval and max e^2: block-wide min/max (exact, order-free)
        double gl = DBL_MAX, gu = -DBL_MAX, emax2 = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const double r = (i > 0 ? fabs(eg[i - 1]) : 0.0) + (i + 1 < n ? fabs(eg[i]) : 0.0);
            const double di = dg[i];
            gl = fmin(gl, di - r);
            gu = fmax(gu, di + r);
            if (i + 1 < n) emax2 = fmax(emax2, eg[i] * eg[i]);
        }
        for (int o = 16; o > 0; o >>= 1) {
            gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
            gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
            emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
        }
        if ((threadIdx.x & 31) == 0) {
            red3[0][threadIdx.x >> 5] = gl;
            red3[1][threadIdx.x >> 5] = gu;
            red3[2][threadIdx.x >> 5] = emax2;
        }
    }
    if (blockIdx.x == 0) {  // ||T||_inf = max_i |d_i| + |e_i-1| + |e_i| for eig_vectors' tolerances
        double rn = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            rn = fmax(rn, fabs(dg[i]) + (i > 0 ? fabs(eg[i - 1]) : 0.0) + (i + 1 < n ? fabs(eg[i]) : 0.0));
        for (int o = 16; o > 0; o >>= 1) rn = fmax(rn, __shfl_xor_sync(0xffffffffu, rn, o));
        if ((threadIdx.x & 31) == 0) red3[0][16 + (threadIdx.x >> 5)] = rn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0) {
            double rn = 0.0;
            for (int w2 = 0; w2 < static_cast<int>(blockDim.x >> 5); ++w2) rn = fmax(rn, red3[0][16 + w2]);
            evals_desc[n] = rn;
        }
        double gl = DBL_MAX, gu = -DBL_MAX, emax2 = 0.0;
        for (int w2 = 0; w2 < static_cast<int>(blockDim.x >> 5); ++w2) {
            gl = fmin(gl, red3[0][w2]);
            gu = fmax(gu, red3[1][w2]);
            emax2 = fmax(emax2, red3[2][w2]);
        }
        const double tnorm = fmax(fabs(gl), fabs(gu));
        const double pivmin = DBL_MIN * fmax(1.0, emax2);
        bounds[0] = gl - 2.0 * DBL_EPSILON * tnorm * n - 2.0 * pivmin;
        bounds[1] = gu + 2.0 * DBL_EPSILON * tnorm * n + 2.0 * pivmin;
        bounds[2] = pivmin;
        // power of two >= ||T|| (exact scaling of d, e^2 and the probes)
        bounds[3] = tnorm > 0.0 ? __longlong_as_double(static_cast<long long>(1023 - dexp(tnorm) - 1) << 52) : 1.0;
    }
    __syncthreads();
    const double inv_sc = bounds[3];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        d[i] = dg[i] * inv_sc;
        if (i + 1 < n) e2[i] = (eg[i] * inv_sc) * (eg[i] * inv_sc);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (j >= n) return;
    constexpr int NP = 32 * kProbes;
    double lo = bounds[0], hi = bounds[1];
    const double pivmin = bounds[2];
    auto probe = [&](int idx) {
        return fmin(fmax(lo + (hi - lo) * (static_cast<double>(idx + 1) / (NP + 1)), lo), hi);
    };
    for (int it = 0; it < 20; ++it) {
        if (!(hi - lo > 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + pivmin)) break;
        double x[kProbes];
        int c[kProbes];
#pragma unroll
        for (int u = 0; u < kProbes; ++u) x[u] = probe(kProbes * lane + u) * inv_sc;
        bool hit;
        sturm_poly<kProbes>(d, e2, n, x, c, hit);
        if (hit) {
#pragma unroll
            for (int u = 0; u < kProbes; ++u) c[u] = sturm_ratio(d, e2, n, x[u], pivmin * inv_sc * inv_sc);
        }
        unsigned mk = 0;
#pragma unroll
        for (int u = 0; u < kProbes; ++u) mk |= (c[u] > j ? 1u : 0u) << u;
        const unsigned ball = __ballot_sync(0xffffffffu, mk != 0);
        int first = NP;
        if (ball) {
            const int fl = __ffs(ball) - 1;
            const unsigned fm = __shfl_sync(0xffffffffu, mk, fl);
            first = kProbes * fl + __ffs(fm) - 1;
        }
        const double nhi = first < NP ? probe(first) : hi;
        const double nlo = first > 0 ? probe(first - 1) : lo;
        if (nlo == lo && nhi == hi) break;
        lo = nlo;
        hi = nhi;
    }
    if (lane == 0) evals_desc[n - 1 - j] = 0.5 * (lo + hi);
}

// ---------------------------------------------------------------- eigenvectors
__device__ __forceinline__ double hash_unit(unsigned a, unsigned b) {
    unsigned h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    h *= 0x297A2D39u;
    h ^= h >> 15;
    return (static_cast<double>(h) / 4294967295.0) * 2.0 - 1.0;
}

// Inverse iteration for eigenvalue j (one CTA of 32 threads per vector).
// shift[j] is the (cluster-perturbed) eigenvalue; Z column-major n x r.
__global__ void __launch_bounds__(32) invit_kernel(const double* __restrict__ dg, const double* __restrict__ eg, int n,
                                                   const double* __restrict__ shift, double tol,
                                                   double* __restrict__ Z) {
    extern __shared__ double sh_inv[];
    double* a = sh_inv;      // U diagonal reciprocal
    double* b = a + n;       // first superdiagonal
    double* c = b + n;       // multipliers
    double* dd = c + n;      // second superdiagonal
    double* x = dd + n;      // iterate
    int* piv = reinterpret_cast<int*>(x + n);
    const int j = blockIdx.x;
    const double lam = shift[j];
    // stage T - lam I (a: diagonal, b: superdiagonal, c: subdiagonal) with all lanes
    for (int i = threadIdx.x; i < n; i += 32) {
        a[i] = dg[i] - lam;
        b[i] = i + 1 < n ? eg[i] : 0.0;
        c[i] = b[i];
        dd[i] = 0.0;
        x[i] = hash_unit(static_cast<unsigned>(j) + 1u, i);
    }
    __syncwarp();
    auto tolfix = [&](double v) { return fabs(v) < tol ? (v < 0.0 ? -tol : tol) : v; };
    if (threadIdx.x == 0) {
        // LU with partial pivoting (LAPACK dlagtf scheme); the updated a[k+1]
        // and b[k+1] ride in registers, a[] receives the pivots' reciprocals
        double ak = a[0], bk = b[0];
        for (int k = 0; k + 1 < n; ++k) {
            const double ck = c[k], an = a[k + 1], bn = b[k + 1];
            if (fabs(ak) >= fabs(ck)) {
                ak = tolfix(ak);
                const double mult = ck * frcp(ak);
                c[k] = mult;
                piv[k] = 0;
                a[k] = frcp(ak);
                b[k] = bk;
                ak = an - mult * bk;
                bk = bn;
            } else {
                const double mult = ak * frcp(ck);
                a[k] = frcp(tolfix(ck));
                b[k] = an;
                c[k] = mult;
                piv[k] = 1;
                const double d2 = k + 2 < n ? bn : 0.0;
                dd[k] = d2;
                ak = bk - mult * an;
                bk = k + 2 < n ? -mult * d2 : bn;
            }
        }
        a[n - 1] = frcp(tolfix(ak));
        b[n - 1] = bk;
    }
    __syncwarp();
    for (int it = 0; it < 3; ++it) {
        if (threadIdx.x == 0) {
            // forward: the carried x[k] stays in a register
            double xk = x[0];
            for (int k = 0; k + 1 < n; ++k) {
                const double xn = x[k + 1], ck = c[k];
                if (piv[k]) {
                    x[k] = xn;
                    xk = xk - ck * xn;
                } else {
                    x[k] = xk;
                    xk = xn - ck * xk;
                }
            }
            x[n - 1] = xk;
            // back substitution with x1 = x[k+1], x2 = x[k+2] in registers
            double x1 = 0.0, x2 = 0.0;
            for (int k = n - 1; k >= 0; --k) {
                double t = (x[k] - b[k] * x1 - dd[k] * x2) * a[k];
                if (fabs(t) > 1e150) {  // rescale the partial solution
                    for (int q = k + 1; q < n; ++q) x[q] *= 1e-150;
                    t *= 1e-150;
                    x1 *= 1e-150;
                }
                x[k] = t;
                x2 = x1;
                x1 = t;
            }
        }
        __syncwarp();
        double s = 0.0;
        for (int i = threadIdx.x; i < n; i += 32) s += x[i] * x[i];
        const double inv = 1.0 / sqrt(warp_sum(s));
        for (int i = threadIdx.x; i < n; i += 32) x[i] *= inv;
        __syncwarp();
    }
    for (int i = threadIdx.x; i < n; i += 32) Z[static_cast<size_t>(j) * n + i] = x[i];
}

// modified Gram-Schmidt inside each tight cluster (one CTA per cluster)
__global__ void cluster_mgs_kernel(const int* __restrict__ clusters, int n, double* __restrict__ Z) {
    __shared__ double red[32];
    const int j0 = clusters[2 * blockIdx.x], j1 = clusters[2 * blockIdx.x + 1];
    for (int j = j0; j < j1; ++j) {
        double* zj = Z + static_cast<size_t>(j) * n;
        for (int pass = 0; pass < 2; ++pass)
            for (int q = j0; q < j; ++q) {
                const double* zq = Z + static_cast<size_t>(q) * n;
                double dt = 0.0;
                for (int i = threadIdx.x; i < n; i += blockDim.x) dt += zq[i] * zj[i];
                dt = block_sum(dt, red);
                for (int i = threadIdx.x; i < n; i += blockDim.x) zj[i] -= dt * zq[i];
                __syncthreads();
            }
        double s = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) s += zj[i] * zj[i];
        const double inv = 1.0 / sqrt(block_sum(s, red));
        for (int i = threadIdx.x; i < n; i += blockDim.x) zj[i] *= inv;
        __syncthreads();
    }
}

// ---------------------------------------------------------------- large clusters
// A cluster of k > 32 inverse-iteration vectors (rows j0..j1 of Z) is
// orthonormalised by CholQR2 instead of MGS (MGS costs 2k^2 dependent dot
// products, ~150 ms for the 468-vector noise-floor cluster of a 500-row mode):
// C = Z_c Z_c^T (the SYRK kernel), an elimination-form Cholesky of C with the
// inverse accumulated (E = L^-1, C = L D L^T; one launch per pivot, the
// trailing update spread over the GPU), Z_c <- D^-1/2 E Z_c (the TTM kernel);
// twice.  Like MGS it keeps the nested spans of the vectors in order; a
// non-positive pivot falls back to MGS for that cluster.
// All k elimination steps in one cooperative launch (one grid barrier per step
// instead of one launch per step); C and E live in L2 (read with ld.cg: other
// CTAs wrote them in earlier steps).  Elimination form: step j takes the Schur
// complement of C below pivot j and accumulates E = L^-1 (C = L D L^T) beside it.
__global__ void __launch_bounds__(256) bigchol_coop_kernel(double* __restrict__ C, double* __restrict__ E,
                                                           double* __restrict__ rinv, int k, int* __restrict__ bad,
                                                           unsigned* __restrict__ ctr) {
    unsigned phase = 0;
    const u64 kk = static_cast<u64>(k) * k;
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    const u64 t0 = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (u64 e = t0; e < kk; e += stride) E[e] = (e / k) == (e % k) ? 1.0 : 0.0;
    coop_barrier(ctr, phase);
    for (int j = 0; j < k; ++j) {
        const double djj = __ldcg(C + static_cast<u64>(j) * k + j);
        if (!(djj >= DBL_MIN)) {
            if (t0 == 0) *bad = 1;
            return;  // every CTA reads the same pivot: all leave here
        }
        const double ri = rsqrt(djj), inv = ri * ri;
        if (t0 == 0) rinv[j] = ri;
        const u64 m = static_cast<u64>(k - j - 1);
        const u64 nc = m, ne = static_cast<u64>(j + 1);
        const u64 total = m * (nc + ne);
        const double* rowj = C + static_cast<u64>(j) * k;
        const double* erow = E + static_cast<u64>(j) * k;
        for (u64 e = t0; e < total; e += stride) {
            const u64 i = j + 1 + e / (nc + ne), c = e % (nc + ne);
            const double f = __ldcg(rowj + i) * inv;
            if (c < nc) {
                const u64 col = j + 1 + c;
                C[i * k + col] = fma(-f, __ldcg(rowj + col), __ldcg(C + i * k + col));
            } else {
                const u64 col = c - nc;
                E[i * k + col] = fma(-f, __ldcg(erow + col), __ldcg(E + i * k + col));
            }
        }
        coop_barrier(ctr, phase);
    }
}

// W[m][c] = E[c][m] rinv[c]  (so that Z_c^T W = (D^-1/2 E Z_c)^T)
__global__ void bigchol_w_kernel(const double* __restrict__ E, const double* __restrict__ rinv, int k,
                                 double* __restrict__ W) {
    const u64 kk = static_cast<u64>(k) * k;
    for (u64 e = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; e < kk; e += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u64 m = e / k, c = e % k;
        W[e] = c >= m ? E[c * k + m] * rinv[c] : 0.0;
    }
}

// true on success; Zc (k rows of length n) orthonormalised in place
bool cluster_cholqr2(double* Zc, int n, int k, cudaStream_t s) {
    DevBuf<double> C(static_cast<u64>(k) * k, s), E(static_cast<u64>(k) * k, s), W(static_cast<u64>(k) * k, s);
    DevBuf<double> rinv(k, s), out(static_cast<u64>(n) * k, s);
    DevBuf<int> bad(1, s);
    bad.zero();
    for (int pass = 0; pass < 2; ++pass) {
        gram_f64(Zc, static_cast<u64>(k), static_cast<u64>(n), C.p, s);
        {
            DevBuf<unsigned> ctr(1, s);
            ctr.zero();
            const unsigned grid = std::min<unsigned>(static_cast<unsigned>(sm_count()),
                                                     cdiv(static_cast<u64>(k) * k, 256));
            double* cp = C.p;
            double* ep = E.p;
            double* rp = rinv.p;
            int* bp = bad.p;
            unsigned* cq = ctr.p;
            int kv = k;
            void* args[] = {&cp, &ep, &rp, &kv, &bp, &cq};
            TCB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bigchol_coop_kernel), dim3(grid), dim3(256),
                                                 args, 0, s));
        }
        bigchol_w_kernel<<<grid_for(static_cast<u64>(k) * k, 256, 4, 4), 256, 0, s>>>(E.p, rinv.p, k, W.p);
        ttm_f64(Zc, static_cast<u64>(k), static_cast<u64>(n), W.p, static_cast<u64>(k), out.p, s);  // n x k
        permute_axes(out.p, Zc, std::vector<u64>{static_cast<u64>(n), static_cast<u64>(k)},
                     std::vector<u64>{1, 0}, s);
        count_launch(3);
    }
    TCB_LAUNCH();
    return bad.to_host()[0] == 0;
}

// ---------------------------------------------------------------- back-transform
// U = Q Z with Q = H_0 ... H_{n-3} (the Gram's eigenvectors from those of the
// tridiagonal, sthosvd.cpp:80-90).  Reflector chunks of KC (32 / 16 / 8 for
// n <= 256 / 512 / 1024) are listed from the last reflector down: chunk c is
// [lo, hi], hi = n-3-c*KC, lo = max(0, hi-KC+1).  H_lo ... H_hi = I - Y T Y^T
// with Y's column q = reflector lo+q (zero above row lo+q+1) and T upper
// triangular: T_jj = tau_j, T[0:j, j] = -tau_j T[0:j, 0:j] (Y^T Y)[0:j, j].
//   wy_tmat : one CTA per chunk (chunks are independent) -> T to global;
//   wy_apply: Z <- Z - Y (T (Y^T Z)) for the chunks in order, one CTA per ZC
//             columns of Z, the next chunk's Y streaming in by cp.async while
//             the current one is applied.  Y^T Z and Y W are 4x4
//             register-blocked; Y^T Z splits the rows over interleaved slices.
constexpr int kBtThreads = 256;

__device__ __forceinline__ void cp_async8_zfill(void* smem, const void* gmem, bool valid) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0));
}

// Yt[q][i] (row stride n + 1) = V[(lo+q) n + i] for i >= lo+q+1 and q < kc, else 0
__device__ __forceinline__ void bt_load_chunk(double* Yt, const double* __restrict__ V, int n, int lo, int kc,
                                              int KC) {
    const int ld = n + 1;
    for (int idx = threadIdx.x; idx < KC * n; idx += blockDim.x) {
        const int q = idx / n, i = idx - q * n;
        const bool valid = q < kc && i >= lo + q + 1;
        cp_async8_zfill(Yt + q * ld + i, V + (valid ? static_cast<size_t>(lo + q) * n + i : 0), valid);
    }
    asm volatile("cp.async.commit_group;\n");
}

__global__ void __launch_bounds__(kBtThreads) wy_tmat(const double* __restrict__ V, const double* __restrict__ tau,
                                                     int n, int KC, double* __restrict__ Tg) {
    extern __shared__ double sbt[];
    const int ld = n + 1, ts = KC + 1;
    const int c = blockIdx.x;
    const int hi = n - 3 - c * KC, lo = max(0, hi - KC + 1), kc = hi - lo + 1;
    double* Yt = sbt;            // KC x ld
    double* S = Yt + KC * ld;    // KC x ts
    double* T = S + KC * ts;     // KC x ts
    bt_load_chunk(Yt, V, n, lo, kc, KC);
    asm volatile("cp.async.wait_group 0;\n");
    __syncthreads();
    for (int e = threadIdx.x; e < KC * KC; e += blockDim.x) {  // S = Y^T Y, upper part
        const int a = e / KC, b = e % KC;
        double s0 = 0.0, s1 = 0.0;
        if (a <= b && b < kc) {
            const double* ya = Yt + a * ld;
            const double* yb = Yt + b * ld;
            int i = lo + b + 1;
            for (; i + 1 < n; i += 2) {
                s0 = fma(ya[i], yb[i], s0);
                s1 = fma(ya[i + 1], yb[i + 1], s1);
            }
            if (i < n) s0 = fma(ya[i], yb[i], s0);
        }
        S[a * ts + b] = s0 + s1;
        T[a * ts + b] = 0.0;
    }
    __syncthreads();
    for (int j = 0; j < kc; ++j) {
        const double tj = tau[lo + j];
        if (static_cast<int>(threadIdx.x) < j) {
            const int i = threadIdx.x;
            double acc = 0.0;
            for (int l = i; l < j; ++l) acc = fma(T[i * ts + l], S[l * ts + j], acc);
            T[i * ts + j] = -tj * acc;
        }
        if (threadIdx.x == 0) T[j * ts + j] = tj;
        __syncthreads();
    }
    for (int e = threadIdx.x; e < KC * KC; e += blockDim.x)
        Tg[static_cast<size_t>(c) * KC * KC + e] = T[(e / KC) * ts + e % KC];
}

// One CTA per 4 columns of Z.  W = Y^T Z: thread (slice, 4-row q block) sums
// rows i = slice (mod nslice) into a 4x4 register block, pairs of adjacent
// slices combine by shuffles; Z -= Y (T W): one row per thread.
__global__ void __launch_bounds__(kBtThreads) wy_apply(const double* __restrict__ V, const double* __restrict__ Tg,
                                                      int n, int r, int KC, int nchunks,
                                                      const double* __restrict__ Z, double* __restrict__ U) {
    constexpr int ZC = 4;
    extern __shared__ __align__(16) double sbt[];
    const int ld = n + 1;
    const int nblk = KC / 4, nslice = kBtThreads / nblk;
    double* Ybuf = sbt;                          // 2 x KC x ld
    double* Tb = Ybuf + 2 * KC * ld;             // 2 x KC x KC
    double* Zs = Tb + 2 * KC * KC;               // n x 4
    double* part = Zs + n * ZC;                  // (nslice / 4) x KC x 4
    double* Wm = part + (nslice / 4) * KC * ZC;  // KC x 4
    double* W2 = Wm + KC * ZC;                   // KC x 4
    const int c0 = blockIdx.x * ZC;
    const int nc = min(ZC, r - c0);
    for (int i = threadIdx.x; i < n; i += blockDim.x)
#pragma unroll
        for (int c = 0; c < ZC; ++c) Zs[i * ZC + c] = c < nc ? Z[static_cast<size_t>(c0 + c) * n + i] : 0.0;
    auto bounds = [&](int c, int& lo, int& kc) {
        const int hi = n - 3 - c * KC;
        lo = max(0, hi - KC + 1);
        kc = hi - lo + 1;
    };
    auto load = [&](int c) {  // chunk c's reflectors (zero-filled) and T, one cp.async group
        int lo, kc;
        bounds(c, lo, kc);
        double* Yt = Ybuf + (c & 1) * KC * ld;
        for (int q = 0; q < KC; ++q) {
            const double* src = V + static_cast<size_t>(lo + q) * n;
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const bool valid = q < kc && i >= lo + q + 1;
                cp_async8_zfill(Yt + q * ld + i, valid ? src + i : V, valid);
            }
        }
        double* Tc = Tb + (c & 1) * KC * KC;
        for (int e = threadIdx.x; e < KC * KC; e += blockDim.x)
            cp_async8_zfill(Tc + e, Tg + static_cast<size_t>(c) * KC * KC + e, true);
        asm volatile("cp.async.commit_group;\n");
    };
    if (nchunks > 0) load(0);
    const int t = threadIdx.x;
    const int slice = t % nslice, qb = (t / nslice) * 4;
    for (int c = 0; c < nchunks; ++c) {
        int lo, kc;
        bounds(c, lo, kc);
        if (c + 1 < nchunks) {
            load(c + 1);
            asm volatile("cp.async.wait_group 1;\n");
        } else {
            asm volatile("cp.async.wait_group 0;\n");
        }
        __syncthreads();
        const double* Yt = Ybuf + (c & 1) * KC * ld;
        const double* Tc = Tb + (c & 1) * KC * KC;
        const int i0 = lo + 1;  // Y is zero above row lo + 1
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
        for (int i = i0 + slice; i < n; i += nslice) {
            const double2 z01 = *reinterpret_cast<const double2*>(Zs + i * ZC);
            const double2 z23 = *reinterpret_cast<const double2*>(Zs + i * ZC + 2);
            const double z[4] = {z01.x, z01.y, z23.x, z23.y};
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const double y = Yt[(qb + a) * ld + i];
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = fma(y, z[b], acc[a][b]);
            }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                double v = acc[a][b];
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                if ((slice & 3) == 0) part[((slice >> 2) * KC + qb + a) * ZC + b] = v;
            }
        __syncthreads();
        for (int e = t; e < KC * ZC; e += blockDim.x) {
            double v = 0.0;
            for (int s4 = 0; s4 < nslice / 4; ++s4) v += part[s4 * KC * ZC + e];
            Wm[e] = v;
        }
        __syncthreads();
        for (int e = t; e < KC * ZC; e += blockDim.x) {  // W2 = T W (T upper)
            const int q = e / ZC, cc = e % ZC;
            double v = 0.0;
            for (int l = q; l < kc; ++l) v = fma(Tc[q * KC + l], Wm[l * ZC + cc], v);
            W2[e] = v;
        }
        __syncthreads();
        for (int i = i0 + t; i < n; i += blockDim.x) {  // Z -= Y W2, one row per thread
            double u[4] = {0.0, 0.0, 0.0, 0.0};
            for (int q = 0; q < kc; ++q) {
                const double y = Yt[q * ld + i];
#pragma unroll
                for (int b = 0; b < 4; ++b) u[b] = fma(y, W2[q * ZC + b], u[b]);
            }
            double2* zr = reinterpret_cast<double2*>(Zs + i * ZC);
            const double2 z01 = zr[0], z23 = zr[1];
            zr[0] = make_double2(z01.x - u[0], z01.y - u[1]);
            zr[1] = make_double2(z23.x - u[2], z23.y - u[3]);
        }
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < n * nc; idx += blockDim.x) {
        const int i = idx / nc, c = idx % nc;
        U[static_cast<size_t>(i) * r + c0 + c] = Zs[i * ZC + c];
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
__global__ void scale_cols_kernel(double* __restrict__ U, int n, int r, const double* __restrict__ sigma) {
    const u64 total = static_cast<u64>(n) * r;
    for (u64 e = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<u64>(gridDim.x) * blockDim.x) {
        const double sg = sigma[e % r];
        if (sg > 0.0) U[e] /= sg;
    }
}

// Modified Gram-Schmidt with reorthogonalisation (a vanishing column is
// replaced by the first unit vector that survives).  With `skip`, it runs only
// if the CholQR pass before it reported a failure (*skip != 0).
__global__ void mgs_kernel(double* __restrict__ U, int n, int r, const int* __restrict__ skip) {
    if (skip && *skip == 0) return;
    extern __shared__ double sh_mgs[];
    double* red = sh_mgs;
    for (int j = 0; j < r; ++j) {
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

namespace {
constexpr size_t kEigSmemMax = 227 * 1024;
constexpr int kEigMaxN = 2300;  // the compact-WY panels of the back-transform at kc = 4
size_t wy_tmat_smem(int n, int kc) {
    return (static_cast<size_t>(kc) * (n + 1) + 2 * kc * (kc + 1)) * sizeof(double);
}
size_t wy_apply_smem(int n, int kc) {
    const int nslice = kBtThreads / (kc / 4);
    return (2 * static_cast<size_t>(kc) * (n + 1) + 2 * kc * kc + static_cast<size_t>(n) * 4 +
            static_cast<size_t>(nslice / 4 + 2) * kc * 4) * sizeof(double);
}
size_t invit_smem(int n) { return 5 * static_cast<size_t>(n) * sizeof(double) + n * sizeof(int); }
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    SideStream() {
        TCB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        TCB_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        TCB_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    }
};
SideStream& side_stream() {  // one per host thread and device
    static thread_local std::vector<SideStream*> per_dev;
    int dev = 0;
    TCB_CUDA(cudaGetDevice(&dev));
    if (per_dev.size() <= static_cast<size_t>(dev)) per_dev.resize(dev + 1, nullptr);
    if (!per_dev[dev]) per_dev[dev] = new SideStream();
    return *per_dev[dev];
}
}  // namespace

// the whole-GPU tridiagonalisation (false: not co-resident, use the cluster kernel)
bool coop_tridiag(double* A, int n, double* d, double* e, double* V, double* tau, double* P, cudaStream_t s) {
    if (std::getenv("TCB_TRIDIAG_CLUSTER")) return false;
    int dev = 0, coop = 0;
    TCB_CUDA(cudaGetDevice(&dev));
    TCB_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    if (!coop) return false;
    // shared-memory-resident rows when they fit (TCB_TRIDIAG_L2=1: the L2 variant)
    {
        const int G = std::min(sm_count(), n);
        const int Q = (n + G - 1) / G;
        const int S = std::max(1, (kCoopThreads / 32) / Q);
        const size_t smem = (static_cast<size_t>(Q) * n + 4 * static_cast<size_t>(n) + 32 + Q * S) * sizeof(double);
        if (smem <= 220 * 1024 && !std::getenv("TCB_TRIDIAG_L2")) {
            TCB_ONCE_PER_DEVICE(cudaFuncSetAttribute(tridiag_coop_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     220 * 1024));
            int per_sm = 0;
            TCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tridiag_coop_smem, kCoopThreads, smem));
            if (per_sm >= 1) {
                DevBuf<unsigned> ctr(1, s);
                DevBuf<int> flags(n, s);
                ctr.zero();
                flags.zero();
                int q = Q, sg = S, nn = n;
                void* args[] = {&A, &nn, &d, &e, &V, &tau, &P, &ctr.p, &flags.p, &q, &sg};
                TCB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(tridiag_coop_smem), dim3(G),
                                                     dim3(kCoopThreads), args, smem, s));
                count_launch();
                return true;
            }
        }
    }
    const size_t smem = (4 * static_cast<size_t>(n) + 32) * sizeof(double);
    if (smem > 220 * 1024) return false;
    TCB_CUDA(cudaFuncSetAttribute(tridiag_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;
    TCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tridiag_coop, kCoopThreads, smem));
    if (per_sm < 1) return false;
    int G = std::min(sm_count(), n);
    DevBuf<unsigned> ctr(1, s);
    DevBuf<int> flags(n, s);
    ctr.zero();
    flags.zero();
    void* args[] = {&A, &n, &d, &e, &V, &tau, &P, &ctr.p, &flags.p};
    TCB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(tridiag_coop), dim3(G), dim3(kCoopThreads), args,
                                         smem, s));
    count_launch();
    return true;
}

std::vector<double> eig_values(const double* A, u64 n64, EigWork& w, cudaStream_t s) {
    ProfScope prof_scope(kEig, s);
    const int n = static_cast<int>(n64);
    // reflector chunk width of the compact-WY back-transform: the preferred width,
    // narrowed until its shared-memory panels fit (larger modes)
    int kc = n <= 256 ? 32 : n <= 512 ? 16 : 8;
    while (kc > 4 && std::max(wy_tmat_smem(n, kc), wy_apply_smem(n, kc)) > kEigSmemMax) kc /= 2;
    if (std::max(wy_tmat_smem(n, kc), wy_apply_smem(n, kc)) > kEigSmemMax ||
        invit_smem(n) > kEigSmemMax || (4 * static_cast<size_t>(n) + 32) * sizeof(double) > kEigSmemMax)
        throw Error("sthosvd: device eigensolver supports mode sizes up to " + std::to_string(kEigMaxN));
    TCB_ONCE_PER_DEVICE({
        cudaFuncSetAttribute(multisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kEigSmemMax);
        cudaFuncSetAttribute(invit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kEigSmemMax);
    });
    w.n = n64;
    w.d = DevBuf<double>(n64, s);
    w.e = DevBuf<double>(n64 + 1, s);
    w.tau = DevBuf<double>(n64 + 1, s);
    w.evals = DevBuf<double>(n64 + 1, s);  // + ||T||_inf (multisect block 0)
    w.z = DevBuf<double>(n64 * n64, s);  // Householder vectors
    w.tau.zero();
    w.e.zero();
    if (n == 1) {
        TCB_CUDA(cudaMemcpyAsync(w.d.p, A, sizeof(double), cudaMemcpyDeviceToDevice, s));
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kCluster);
        cfg.blockDim = dim3(kTriThreads);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = kCluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        bool dsmem = false;
        if (n <= kDsmemMaxN) {
            const int nloc = (n + kTdCluster - 1) / kTdCluster;
            const size_t smem = ((static_cast<size_t>(nloc) * n + 1) / 2 * 2 + 6 * n) * sizeof(double);
            TCB_ONCE_PER_DEVICE({
                cudaFuncSetAttribute(tridiag_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
                cudaFuncSetAttribute(tridiag_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            });
            cfg.gridDim = dim3(kTdCluster);
            // one row slot per warp up to n = 256, two beyond (fewer redundant per-warp steps)
            cfg.blockDim = dim3(32 * (nloc <= 16 ? nloc : (nloc + 1) / 2));
            at[0].val.clusterDim.x = kTdCluster;
            cfg.dynamicSmemBytes = smem;
            int ncl = 0;  // a 16-CTA cluster with this much shared memory must fit one GPC
            const cudaError_t qe = cudaOccupancyMaxActiveClusters(&ncl, tridiag_dsmem, &cfg);
            dsmem = qe == cudaSuccess && ncl > 0;
            if (std::getenv("TCB_DEBUG"))
                std::fprintf(stderr, "tridiag_dsmem n=%d smem=%zu clusters=%d err=%s\n", n, smem, ncl,
                             cudaGetErrorString(qe));
            cudaGetLastError();
            if (dsmem) TCB_CUDA(cudaLaunchKernelEx(&cfg, tridiag_dsmem, A, n, w.d.p, w.e.p, w.z.p, w.tau.p));
        }
        if (!dsmem) {
            w.a = DevBuf<double>(n64 * n64, s);
            DevBuf<double> P(n64, s);
            TCB_CUDA(cudaMemcpyAsync(w.a.p, A, n64 * n64 * sizeof(double), cudaMemcpyDeviceToDevice, s));
            if (!coop_tridiag(w.a.p, n, w.d.p, w.e.p, w.z.p, w.tau.p, P.p, s)) {
                cfg.gridDim = dim3(kCluster);
                cfg.blockDim = dim3(kTriThreads);
                at[0].val.clusterDim.x = kCluster;
                cfg.dynamicSmemBytes = (2 * n + 32) * sizeof(double);
                TCB_CUDA(cudaLaunchKernelEx(&cfg, tridiag_global, w.a.p, n, w.d.p, w.e.p, w.z.p, w.tau.p, P.p));
            }
        }
        count_launch();
    }
    // compact-WY T matrices of the reflector chunks on a side stream, overlapping the multisection
    w.kc = kc;
    w.nchunks = n >= 3 ? (n - 2 + w.kc - 1) / w.kc : 0;
    w.tg = DevBuf<double>(static_cast<u64>(std::max(w.nchunks, 1)) * w.kc * w.kc, s);
    SideStream& side = side_stream();
    if (w.nchunks > 0) {
        TCB_ONCE_PER_DEVICE(cudaFuncSetAttribute(wy_tmat, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        TCB_CUDA(cudaEventRecord(side.fork, s));
        TCB_CUDA(cudaStreamWaitEvent(side.s, side.fork, 0));
        const size_t tsm = wy_tmat_smem(n, w.kc);
        wy_tmat<<<static_cast<unsigned>(w.nchunks), kBtThreads, tsm, side.s>>>(w.z.p, w.tau.p, n, w.kc, w.tg.p);
        count_launch();
        TCB_CUDA(cudaEventRecord(side.join, side.s));
    }
    const int wpb = 2;
    multisect_kernel<<<cdiv(n64, wpb), 32 * wpb, 2 * n * sizeof(double), s>>>(w.d.p, w.e.p, n, w.evals.p);
    count_launch();
    if (w.nchunks > 0) TCB_CUDA(cudaStreamWaitEvent(s, side.join, 0));
    TCB_LAUNCH();
    std::vector<double> ev(n64 + 1);
    w.evals.download(ev.data(), n64 + 1);  // one synchronising copy: eigenvalues and ||T||_inf
    stream_sync(s);
    w.tnorm = ev[n64];
    ev.resize(n64);
    w.ev = ev;
    return ev;
}

void eig_vectors(EigWork& w, u64 r64, double* U, cudaStream_t s) {
    ProfScope prof_scope(kEig, s);
    const int n = static_cast<int>(w.n), r = static_cast<int>(r64);
    const std::vector<double>& ev = w.ev;  // host copies made by eig_values: no round trip here
    double tnorm = w.tnorm;
    if (!(tnorm > 0.0)) tnorm = 1.0;  // zero matrix: any orthonormal basis is an eigenbasis
    // tight clusters: consecutive eigenvalues closer than 1e-6 ||T||; their
    // vectors are orthogonalised against each other after inverse iteration
    const double ctol = 1e-6 * tnorm;
    std::vector<double> shift(r);
    std::vector<int> clusters;
    int start = 0;
    for (int j = 0; j < r; ++j) {
        shift[j] = ev[j];
        if (j > 0 && ev[j - 1] - ev[j] <= ctol) {
            const double pertol = 10.0 * DBL_EPSILON * std::fabs(ev[j]);
            if (shift[j - 1] - shift[j] < pertol) shift[j] = shift[j - 1] - pertol;
        } else {
            if (j - start >= 2) {
                clusters.push_back(start);
                clusters.push_back(j);
            }
            start = j;
        }
    }
    if (r - start >= 2) {
        clusters.push_back(start);
        clusters.push_back(r);
    }
    DevBuf<double> dsh(r, s);
    dsh.upload(shift.data(), r);
    DevBuf<double> Z(static_cast<u64>(n) * r, s);
    const size_t smem = invit_smem(n);
    invit_kernel<<<static_cast<unsigned>(r), 32, smem, s>>>(w.d.p, w.e.p, n, dsh.p, DBL_EPSILON * tnorm, Z.p);
    count_launch();
    if (!clusters.empty()) {
        // big clusters by CholQR2 (MGS where it breaks down), the rest by MGS
        std::vector<int> small;
        for (std::size_t c = 0; c < clusters.size(); c += 2) {
            const int j0 = clusters[c], j1 = clusters[c + 1], k = j1 - j0;
            bool done = false;
            if (k > 32) {
                DevBuf<double> keep(static_cast<u64>(k) * n, s);
                TCB_CUDA(cudaMemcpyAsync(keep.p, Z.p + static_cast<u64>(j0) * n, keep.n * sizeof(double),
                                         cudaMemcpyDeviceToDevice, s));
                done = cluster_cholqr2(Z.p + static_cast<u64>(j0) * n, n, k, s);
                if (!done)
                    TCB_CUDA(cudaMemcpyAsync(Z.p + static_cast<u64>(j0) * n, keep.p, keep.n * sizeof(double),
                                             cudaMemcpyDeviceToDevice, s));
            }
            if (!done) {
                small.push_back(j0);
                small.push_back(j1);
            }
        }
        if (!small.empty()) {
            DevBuf<int> dcl(small.size(), s);
            dcl.upload(small.data(), small.size());
            cluster_mgs_kernel<<<static_cast<unsigned>(small.size() / 2), 256, 0, s>>>(dcl.p, n, Z.p);
            count_launch();
        }
    }
    // T matrices come from wy_tmat on the side stream (launched by eig_values)
    TCB_ONCE_PER_DEVICE(cudaFuncSetAttribute(wy_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    const int KC = w.kc;
    const size_t asm_ = wy_apply_smem(n, KC);
    wy_apply<<<cdiv(r64, 4), kBtThreads, asm_, s>>>(w.z.p, w.tg.p, n, r, KC, w.nchunks, Z.p, U);
    count_launch();
    TCB_LAUNCH();
}

void fix_column_signs(double* U, u64 n, u64 r, cudaStream_t s) {
    ProfScope prof_scope(kEig, s);
    sign_kernel<<<cdiv(r, 4), 128, 0, s>>>(U, static_cast<int>(n), static_cast<int>(r));
    count_launch();
    TCB_LAUNCH();
}

// U <- orth(U diag(1/sigma)) (the thin branch, sthosvd.cpp:91-99 stand-in): the
// columns are already nearly orthonormal, so shifted CholQR3 on one CTA
// (topk.cu) does it in a few DMMA passes; MGS runs only if that reports a
// Cholesky breakdown (or the panel is too large for it).
void scale_orthonormalize(double* U, u64 n, u64 r, const double* sigma, cudaStream_t s) {
    ProfScope prof_scope(kEig, s);
    scale_cols_kernel<<<grid_for(n * r, 256, 4, 4), 256, 0, s>>>(U, static_cast<int>(n), static_cast<int>(r), sigma);
    DevBuf<int> fail(1, s);
    const bool fast = cholqr_inplace(U, n, static_cast<int>(r), fail.p, s);
    mgs_kernel<<<1, 256, 32 * sizeof(double), s>>>(U, static_cast<int>(n), static_cast<int>(r), fast ? fail.p : nullptr);
    count_launch(2);
    TCB_LAUNCH();
}

}  // namespace tcb

#ifdef TCB_TRIDIAG_TIMING
namespace tcb {
void tri_phase_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_tri_phase, sizeof(unsigned long long) * 160); }
}  // namespace tcb
#endif
