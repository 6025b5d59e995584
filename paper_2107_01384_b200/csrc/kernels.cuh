// Host-callable launchers for every sm_100a kernel of the compress path.
#pragma once

#include <memory>
#include <vector>

#include "common.cuh"

namespace tcb {

// ---- ingest.cu: cast + finite check + ||A||^2 (container.cpp:51-94, kernels_avx2.cpp:68-160)
// dtype codes follow container::Dtype (container.hpp:16-27).
void ingest_cast(const void* src, int dtype, u64 n, double* dst, cudaStream_t s);
void ingest_cast_f32(const void* src, int dtype, u64 n, float* dst, cudaStream_t s);
// Deterministic fixed-tree sum of squares in double; *finite = all elements finite.
double sum_squares(const double* x, u64 n, bool* finite, cudaStream_t s);
double sum_squares(const float* x, u64 n, bool* finite, cudaStream_t s);
// Row-major axis permutation (tensor.cpp:105-144): out axis i = in axis perm[i].
template <class T>
void permute_axes(const T* src, T* dst, const std::vector<u64>& shape, const std::vector<u64>& perm,
                  cudaStream_t s);
// int64/uint64 sources whose magnitude exceeds 2^53 (container.cpp:60-63)
bool ingest_precision_loss(const void* src, int dtype, u64 n, cudaStream_t s);
// sum of (a_i - b_i)^2 (tensor.cpp:147-164); f32 rounds both sides to float first
double sse_between(const double* a, const double* b, u64 n, bool f32, cudaStream_t s);
// trace of an n x n row-major matrix (one round trip)
double gram_trace(const double* G, u64 n, cudaStream_t s);
// max |x| with the all-finite flag, one pass and one round trip
double max_abs_finite(const double* x, u64 n, bool* finite, cudaStream_t s);
// Exact max |x| (kernels_avx2.cpp:40-66 is order-independent, so exact on any tree).
double max_abs(const double* x, u64 n, cudaStream_t s);

// ---- gram.cu: G = B B^T (B row-major rows x cols), fp64 DMMA, deterministic split-K.
// G is written full symmetric, row-major rows x rows.
void gram_f64(const double* B, u64 rows, u64 cols, double* G, cudaStream_t s);
// The same computation in pieces (bitwise identical): the split-K plan, the
// splits [sp0, sp1) (they read only columns [split_col(sp0), split_col(sp1)) of
// B, so they can run as soon as those columns are resident), the fixed-order
// reduction.  gram_f64 = plan + all splits + reduce.
struct GramPlan {
    int lower = 0;
    u64 nslab = 0, per = 0, splits = 0;
    bool v16 = false;
    int variant = 0, bk = 32;  // SYRK kernel shape (gemm.cu kSyrk)
    int n_off = 0, n_diag = 0;  // lower-triangle tiles off / on the diagonal
    u64 per_d = 0, splits_d = 0;  // diagonal tiles' slabs per CTA and split count (per, splits: off-diagonal)
};
GramPlan gram_plan(const double* B, u64 rows, u64 cols);
u64 gram_ws_doubles(const GramPlan& gp);
u64 gram_split_col(const GramPlan& gp, u64 split, u64 cols);
void gram_splits(const double* B, u64 rows, u64 cols, const GramPlan& gp, u64 sp0, u64 sp1, double* ws,
                 cudaStream_t s);
void gram_reduce(const GramPlan& gp, const double* ws, u64 rows, double* G, cudaStream_t s);
// G = B^T B (cols x cols) for the rows > cols branch (sthosvd.cpp:91-99 stand-in).
void gram_cols_f64(const double* B, u64 rows, u64 cols, double* G, cudaStream_t s);

// ---- ttm.cu: out (cols x r, row-major) = B^T U (sthosvd.cpp:158-166), fp64 DMMA.
void ttm_f64(const double* B, u64 rows, u64 cols, const double* U, u64 r, double* out, cudaStream_t s);

// ---- ozaki.cu: the same Gram (full, bitwise symmetric) and TTM by the Ozaki
// scheme on the INT8 tensor cores (5 digit slices, exact int recombination);
// used by the mode loop for shapes where it pays (ozaki_*_ok; TCB_OZAKI=0: never).
bool ozaki_gram_ok(u64 rows, u64 cols);
bool ozaki_ttm_ok(u64 rows, u64 cols, u64 r);
bool ozaki_lt_forced();  // TCB_OZAKI_LT=1: the cuBLASLt cross-check path
void gram_ozaki(const double* B, u64 rows, u64 cols, double* G, cudaStream_t s);
// The same Gram with the rows of B (row-major rows x cols) arriving in order
// (e.g. row slabs of a host upload): rows_ready(B, r1) once rows < r1 are valid
// on s runs their exponents, sums of squares and digits and every product tile
// whose row blocks are complete; finish writes G.  Bitwise gram_ozaki's G (the
// digit products accumulate exactly in int64, the diagonal is per-row).
struct OzGramRows {
    u64 rows, cols, nslab = 0, ra = 0, rb = 0, ld = 0, done = 0;
    cudaStream_t s;
    DevBuf<int> ex;
    DevBuf<double> sq;
    DevBuf<int8_t> da, db;
    DevBuf<long long> acc;
    std::vector<int2> pending;
    OzGramRows(u64 rows, u64 cols, cudaStream_t s);
    void rows_ready(const double* B, u64 r1);
    void finish(double* G);
};
// The TTM's B-side work (column exponents, column digits) depends only on B:
// ttm_ozaki_prepare runs it on `side` (e.g. beside the eigensolve that produces
// U) and ttm_ozaki, given the handle, waits for it instead of redoing it.
struct OzTtmPrep {
    u64 rows = 0, cols = 0, nslab = 0;
    DevBuf<int> exc;
    DevBuf<int8_t> dt;
    cudaEvent_t done = nullptr;
    OzTtmPrep() = default;
    OzTtmPrep(const OzTtmPrep&) = delete;
    OzTtmPrep& operator=(const OzTtmPrep&) = delete;
    ~OzTtmPrep();
};
std::unique_ptr<OzTtmPrep> ttm_ozaki_prepare(const double* B, u64 rows, u64 cols, cudaStream_t side);
void ttm_ozaki(const double* B, u64 rows, u64 cols, const double* U, u64 r, double* out, cudaStream_t s,
               OzTtmPrep* prep = nullptr);
// out (rows x r) = B V  (B rows x cols row-major, V cols x r row-major); small.
void gemm_nn_f64(const double* B, u64 rows, u64 cols, const double* V, u64 r, double* out, cudaStream_t s);

// ---- eig.cu: symmetric eigensolver for n <= 1024 (SelfAdjointEigenSolver stand-in).
struct EigWork {
    DevBuf<double> a;    // n x n working copy (row-major), reflectors below the subdiagonal
    DevBuf<double> d, e, tau, evals, z;
    DevBuf<double> tg;       // compact-WY T matrices, nchunks x kc x kc
    int kc = 0, nchunks = 0;
    std::vector<double> ev;  // host copy of the descending eigenvalues (eig_values)
    double tnorm = 0.0;      // host: ||T||_inf
    u64 n = 0;
};
// Householder tridiagonalisation of the symmetric row-major A (n x n) and
// all eigenvalues by bisection, returned in DESCENDING order (host copy).
std::vector<double> eig_values(const double* A, u64 n, EigWork& w, cudaStream_t s);
// Top-r orthonormal eigenvectors (n x r, row-major) after eig_values.
void eig_vectors(EigWork& w, u64 r, double* U, cudaStream_t s);
// Column sign convention (sthosvd.cpp:103-110): largest |u| (first on ties) >= 0.
void fix_column_signs(double* U, u64 n, u64 r, cudaStream_t s);
// Normalise columns of U (n x r row-major) by 1/sigma_j and re-orthonormalise (MGS).
void scale_orthonormalize(double* U, u64 n, u64 r, const double* sigma, cudaStream_t s);
// In-place shifted CholQR3 of a row-major n x r panel (n <= 256, r <= 32) on one
// CTA; *fail_dev is zeroed and set on a Cholesky breakdown (U then unchanged).
// Returns false (nothing launched) when the panel does not fit.
bool cholqr_inplace(double* U, u64 n, int r, int* fail_dev, cudaStream_t s);

// ---- topk.cu: certified top-p eigenpairs by block subspace iteration + Rayleigh-Ritz.
bool topk_supported(u64 n, int p);
// X (n x p row-major): Ritz vectors for theta (descending); resid[j] = |G x_j - theta_j x_j|;
// trace = trace(G).  Synchronises the stream (host copies of theta / resid / trace).
void topk_eig(const double* G, u64 n, int p, int extra_iters, double* X, std::vector<double>& theta,
              std::vector<double>& resid, double& trace, cudaStream_t s);

// ---- quant.cu (core_codec.cpp:55-93)
// order (optional): the vectorisation map, coefficient v = x[order[v]]
void quantize_f64(const double* x, u64 n, int k, u64* mag, u8* neg, cudaStream_t s, const u64* order = nullptr);
// Per-axis slice sums of (double)m^2 replayed in vectorisation order, then sqrt(s*down).
void slice_norms(const u64* mag, const std::vector<u64>& shape, double down, double* out, cudaStream_t s,
                 const u64* order = nullptr);

}  // namespace tcb
