// fp64 Gram and TTM by the Ozaki scheme on the INT8 tensor cores.
//
// The reference's fp64-internal mode computes X X^T and X^T U in double
// (sthosvd.cpp:78-79, 158-166).  DMMA (mma.sync m8n8k4 f64) tops out at
// ~37 TF/s on B200; the INT8 tensor cores run ~3 POP/s.  Each row of X (and
// each column of U for the TTM) is scaled by a power of two to |x| < 1 and
// split exactly into five digit slices of 6 + 7 + 7 + 7 + 7 bits,
//     x = 2^e sum_s d_s 2^-(6 + 7 s),   d_s in [-64, 64],
// (the digits are exact: every step is a power-of-two scaling and the
// subtraction of a nearby integer), truncating x 34 bits below its row's top.
// Products of digits of slices s and t carry the weight 2^-(12 + 7 (s + t)),
// so all pairs of one level L = s + t are summed by ONE int8 GEMM over the
// slices concatenated along k:  [d_0 .. d_L] . [d'_L .. d'_0]^T.  Levels
// L <= 4 are kept (the dropped levels weigh <= 2^-47 of the row products).
// int32 accumulation is exact (|digit products| <= 2^12, at most 2^15 of them
// per Gram k-chunk, at most 5 * 2300 per TTM dot product), the levels combine
// exactly in int64 as sum_L C_L 2^(7 (4 - L)) (< 2^63), and one rounding to
// double and a power-of-two scale give the result.  The outcome is therefore
// deterministic and independent of the GEMM's summation order; against the
// fp64 Gram of c5 it differs by <= 1.4e-11 |x_i||x_j| (tools/ozaki_eval.py:
// top-650 eigenvalues within 2.6e-14 lambda_1, subspace identical to fp64
// resolution).  The Gram's diagonal is the fp64 row sum of squares.
//
// The digit products run on the tcgen05 tensor cores in ozmma.cu (TMA-staged
// slices, the five level accumulators in tensor memory, exact int64 combine in
// the epilogue).  TCB_OZAKI_LT=1 runs the same products as cuBLASLt IMMA GEMMs
// instead (k-concatenated slices, one GEMM per level): integer results, so the
// two paths agree bit for bit (tests/test_gpu_ozaki.py).
#include <cublasLt.h>

#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "kernels.cuh"
#include "ozmma.cuh"

namespace tcb {

namespace {

constexpr int kSlices = 5;
constexpr u64 kGramKC = u64{1} << 15;  // Gram k-chunk per int32 partial: 2^12 * 2^15 = 2^27

#define TCB_LT(x)                                                                                     \
    do {                                                                                              \
        const cublasStatus_t st_ = (x);                                                               \
        if (st_ != CUBLAS_STATUS_SUCCESS)                                                             \
            throw Error(std::string("cuBLASLt: ") + #x + " failed (" + std::to_string(static_cast<int>(st_)) + ")"); \
    } while (0)

cublasLtHandle_t lt_handle() {
    static PerDevice<cublasLtHandle_t> h;
    return h.get([] {
        cublasLtHandle_t x = nullptr;
        TCB_LT(cublasLtCreate(&x));
        return x;
    });
}

// C (m x n, column-major, ldc, int32) = A^T B, A stored k-contiguous as m rows
// of lda bytes, B as n rows of ldb bytes; `batch` matrices at strides sa/sb/sc.
void imma_tn(const int8_t* A, u64 lda, long long sa, const int8_t* B, u64 ldb, long long sb, int32_t* C, u64 ldc,
             long long sc, u64 m, u64 n, u64 k, int batch, cudaStream_t s) {
    cublasLtHandle_t h = lt_handle();
    cublasLtMatmulDesc_t op = nullptr;
    cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
    cublasLtMatmulPreference_t pref = nullptr;
    struct Guard {
        cublasLtMatmulDesc_t& op;
        cublasLtMatrixLayout_t &la, &lb, &lc;
        cublasLtMatmulPreference_t& pref;
        ~Guard() {
            if (pref) cublasLtMatmulPreferenceDestroy(pref);
            if (lc) cublasLtMatrixLayoutDestroy(lc);
            if (lb) cublasLtMatrixLayoutDestroy(lb);
            if (la) cublasLtMatrixLayoutDestroy(la);
            if (op) cublasLtMatmulDescDestroy(op);
        }
    } guard{op, la, lb, lc, pref};
    TCB_LT(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32I, CUDA_R_32I));
    const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    TCB_LT(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)));
    TCB_LT(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)));
    TCB_LT(cublasLtMatrixLayoutCreate(&la, CUDA_R_8I, k, m, static_cast<int64_t>(lda)));
    TCB_LT(cublasLtMatrixLayoutCreate(&lb, CUDA_R_8I, k, n, static_cast<int64_t>(ldb)));
    TCB_LT(cublasLtMatrixLayoutCreate(&lc, CUDA_R_32I, m, n, static_cast<int64_t>(ldc)));
    if (batch > 1) {
        const int32_t bc = batch;
        const int64_t oa = sa, ob = sb, oc = sc;
        for (auto [l, o] : {std::pair{la, oa}, std::pair{lb, ob}, std::pair{lc, oc}}) {
            TCB_LT(cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc)));
            TCB_LT(cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &o, sizeof(o)));
        }
    }
    const size_t wsz = 32ull << 20;
    TCB_LT(cublasLtMatmulPreferenceCreate(&pref));
    TCB_LT(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof(wsz)));
    // the algorithm per shape, once per device
    using Key = std::tuple<u64, u64, u64, u64, u64, u64, long long, long long, long long, int>;
    static PerDevice<std::map<Key, cublasLtMatmulAlgo_t>> algos;
    static std::mutex mu;
    auto& amap = algos.get([] { return std::map<Key, cublasLtMatmulAlgo_t>{}; });
    const Key key{m, n, k, lda, ldb, ldc, sa, sb, sc, batch};
    cublasLtMatmulAlgo_t algo;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = amap.find(key);
        if (it == amap.end()) {
            cublasLtMatmulHeuristicResult_t res{};
            int nres = 0;
            TCB_LT(cublasLtMatmulAlgoGetHeuristic(h, op, la, lb, lc, lc, pref, 1, &res, &nres));
            if (nres < 1) throw Error("cuBLASLt: no int8 GEMM algorithm for the Ozaki split");
            it = amap.emplace(key, res.algo).first;
        }
        algo = it->second;
    }
    DevBuf<u8> ws(wsz, s);
    const int32_t alpha = 1, beta = 0;
    TCB_LT(cublasLtMatmul(h, op, &alpha, A, la, B, lb, &beta, C, lc, C, lc, &algo, ws.p, wsz, s));
}

__device__ __forceinline__ void digits(double r, int8_t (&d)[kSlices]) {  // |r| < 1
    double v = r * 64.0;
#pragma unroll
    for (int q = 0; q < kSlices; ++q) {
        const double t = rint(v);
        d[q] = static_cast<int8_t>(t);
        v = (v - t) * 128.0;  // exact: |v - t| <= 1/2
    }
}

// per row: exponent e with max|x| < 2^e, and the fp64 sum of squares (fixed tree)
__global__ void __launch_bounds__(256) oz_rowstat_kernel(const double* __restrict__ B, u64 cols, int* __restrict__ ex,
                                                         double* __restrict__ sumsq) {
    __shared__ double smx[8], ssq[8];
    const double* row = B + static_cast<u64>(blockIdx.x) * cols;
    double mx = 0.0, sq = 0.0;
    for (u64 j = threadIdx.x; j < cols; j += blockDim.x) {
        const double x = row[j];
        mx = fmax(mx, fabs(x));
        sq = fma(x, x, sq);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
    }
    if ((threadIdx.x & 31) == 0) {
        smx[threadIdx.x >> 5] = mx;
        ssq[threadIdx.x >> 5] = sq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0, q = 0.0;
        for (int w = 0; w < 8; ++w) {
            m = fmax(m, smx[w]);
            q += ssq[w];
        }
        ex[blockIdx.x] = m > 0.0 ? ilogb(m) + 1 : 0;
        sumsq[blockIdx.x] = q;
    }
}

// per column of a rows x cols matrix: exponent e with max|x| < 2^e
__global__ void oz_colexp_kernel(const double* __restrict__ B, u64 rows, u64 cols, int* __restrict__ ex) {
    const u64 c = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    double mx = 0.0;
    for (u64 k = 0; k < rows; ++k) mx = fmax(mx, fabs(B[k * cols + c]));
    ex[c] = mx > 0.0 ? ilogb(mx) + 1 : 0;
}

// Gram slices: row i of Dcat is [d_0 | d_1 | .. | d_4] and of Drev [d_4 | .. | d_0],
// each slice Kp long (zero beyond cols); 4 consecutive k per thread
__global__ void __launch_bounds__(256) oz_split_rows_kernel(const double* __restrict__ B, u64 cols, u64 Kp,
                                                            const int* __restrict__ ex, int8_t* __restrict__ Dcat,
                                                            int8_t* __restrict__ Drev) {
    const u64 i = blockIdx.y;
    const u64 k0 = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (k0 >= Kp) return;
    const double sc = scalbn(1.0, -ex[i]);
    int8_t d[4][kSlices];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const u64 k = k0 + q;
        const double x = k < cols ? B[i * cols + k] : 0.0;
        digits(x * sc, d[q]);
    }
    const u64 base = i * kSlices * Kp;
#pragma unroll
    for (int s = 0; s < kSlices; ++s) {
        const char4 v = make_char4(d[0][s], d[1][s], d[2][s], d[3][s]);
        *reinterpret_cast<char4*>(Dcat + base + static_cast<u64>(s) * Kp + k0) = v;
        *reinterpret_cast<char4*>(Drev + base + static_cast<u64>(kSlices - 1 - s) * Kp + k0) = v;
    }
}

// TTM slices of a rows x cols matrix, transposed: output row c (< cols_p) holds
// the digits of column c over k < Kr (zero beyond rows), slice order s (rev = 0)
// or 4 - s (rev = 1) in segments of Kr.  32 x 32 tiles through shared memory.
__global__ void __launch_bounds__(256) oz_split_cols_kernel(const double* __restrict__ B, u64 rows, u64 cols,
                                                            u64 cols_p, u64 Kr, const int* __restrict__ ex, int rev,
                                                            int8_t* __restrict__ out) {
    __shared__ int8_t t[kSlices][32][33];
    const u64 c0 = static_cast<u64>(blockIdx.x) * 32, k0 = static_cast<u64>(blockIdx.y) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
    for (int kk = ty; kk < 32; kk += 8) {
        const u64 k = k0 + kk, c = c0 + tx;
        double x = 0.0;
        int e = 0;
        if (c < cols) {
            e = ex[c];
            if (k < rows) x = B[k * cols + c];
        }
        int8_t d[kSlices];
        digits(x * scalbn(1.0, -e), d);
#pragma unroll
        for (int s = 0; s < kSlices; ++s) t[s][tx][kk] = d[s];
    }
    __syncthreads();
    for (int cc = ty; cc < 32; cc += 8) {
        const u64 c = c0 + cc, k = k0 + tx;
        if (c >= cols_p || k >= Kr) continue;
#pragma unroll
        for (int s = 0; s < kSlices; ++s) {
            const int seg = rev ? kSlices - 1 - s : s;
            out[c * kSlices * Kr + static_cast<u64>(seg) * Kr + k] = t[s][cc][tx];
        }
    }
}

// Blocked digit layouts for the tcgen05 path (ozmma.cuh): row i of B split as
// oz_split_rows_kernel does, written into the 128-row and the 96-row blocking
// (rows up to either padding are zero); 4 consecutive k per thread.
__global__ void __launch_bounds__(256) oz_split_rows_blk_kernel(const double* __restrict__ B, u64 rows, u64 cols,
                                                                u64 nslab, const int* __restrict__ ex,
                                                                int8_t* __restrict__ DA, u64 rows_a,
                                                                int8_t* __restrict__ DB, u64 rows_b, u64 i0) {
    const u64 i = i0 + blockIdx.y;
    const u64 k0 = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (k0 >= nslab * kOzSlab) return;
    int8_t d[4][kSlices];
    const double sc = i < rows ? scalbn(1.0, -ex[i]) : 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const u64 k = k0 + q;
        const double x = i < rows && k < cols ? B[i * cols + k] : 0.0;
        digits(x * sc, d[q]);
    }
#pragma unroll
    for (int s = 0; s < kSlices; ++s) {
        const char4 v = make_char4(d[0][s], d[1][s], d[2][s], d[3][s]);
        if (i < rows_a) *reinterpret_cast<char4*>(DA + oz_block_off(i, k0, s, kOzBM, nslab)) = v;
        if (i < rows_b) *reinterpret_cast<char4*>(DB + oz_block_off(i, k0, s, kOzBN, nslab)) = v;
    }
}

// Columns of a rows x cols matrix as rows of the blocked layout (block rows br):
// output row c holds the digits of column c over k < 64 nslab (zero beyond rows
// and for c >= cols up to the padding).  32 columns x 128 k per CTA, through
// shared memory 32 k at a time; each thread writes 4 consecutive k of one
// column per slice.
constexpr int kColK = 128;
__global__ void __launch_bounds__(256) oz_split_cols_blk_kernel(const double* __restrict__ B, u64 rows, u64 cols,
                                                                u64 cols_pad, u64 nslab, const int* __restrict__ ex,
                                                                u32 br, int8_t* __restrict__ out) {
    __shared__ int8_t t[kSlices][32][36];
    const u64 c0 = static_cast<u64>(blockIdx.x) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
    const u64 cr = c0 + tx;
    const double sc = cr < cols ? scalbn(1.0, -ex[cr]) : 0.0;
    const int cc = threadIdx.x >> 3, kq = (threadIdx.x & 7) * 4;
    const u64 cw = c0 + cc;
    for (int sub = 0; sub < kColK / 32; ++sub) {
        const u64 k0 = static_cast<u64>(blockIdx.y) * kColK + sub * 32;
        if (k0 >= nslab * kOzSlab) break;
        for (int kk = ty; kk < 32; kk += 8) {
            const u64 k = k0 + kk;
            const double x = cr < cols && k < rows ? B[k * cols + cr] : 0.0;
            int8_t d[kSlices];
            digits(x * sc, d);
#pragma unroll
            for (int s = 0; s < kSlices; ++s) t[s][tx][kk] = d[s];
        }
        __syncthreads();
        const u64 k = k0 + kq;
        if (cw < cols_pad && k < nslab * kOzSlab) {
#pragma unroll
            for (int s = 0; s < kSlices; ++s) {
                const char4 v = make_char4(t[s][cc][kq], t[s][cc][kq + 1], t[s][cc][kq + 2], t[s][cc][kq + 3]);
                *reinterpret_cast<char4*>(out + oz_block_off(cw, k, s, br, nslab)) = v;
            }
        }
        __syncthreads();
    }
}

struct LevelPtrs {
    const int32_t* c[kSlices];
    int nb[kSlices];
};

// G (rows x rows) from the level partials: C_L batch b is rows_p x rows_p column-major
__global__ void oz_gram_combine_kernel(LevelPtrs lv, u64 rows, u64 rows_p, const int* __restrict__ ex,
                                       const double* __restrict__ sumsq, double* __restrict__ G) {
    const u64 e = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= rows * rows) return;
    const u64 i = e / rows, j = e % rows;
    if (i == j) {
        G[e] = sumsq[i];
        return;
    }
    // the level sums are exactly symmetric (both (s, t) and (t, s) are in a level),
    // so entry (i, j) is read row-wise: consecutive threads, consecutive addresses
    const u64 off = i * rows_p + j, mat = rows_p * rows_p;
    long long T = 0;
#pragma unroll
    for (int L = 0; L < kSlices; ++L) {
        long long s = 0;
        for (int b = 0; b < lv.nb[L]; ++b) s += lv.c[L][static_cast<u64>(b) * mat + off];
        T += s * (1LL << (7 * (kSlices - 1 - L)));
    }
    G[e] = scalbn(static_cast<double>(T), ex[i] + ex[j] - 40);
}

// G from the tensor-core path's int64 accumulator (lower triangle valid)
__global__ void oz_gram_final_kernel(const long long* __restrict__ acc, u64 ld, u64 rows, const int* __restrict__ ex,
                                     const double* __restrict__ sumsq, double* __restrict__ G) {
    const u64 e = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= rows * rows) return;
    const u64 i = e / rows, j = e % rows;
    if (i == j) {
        G[e] = sumsq[i];
        return;
    }
    const long long T = i > j ? acc[i * ld + j] : acc[j * ld + i];
    G[e] = scalbn(static_cast<double>(T), ex[i] + ex[j] - 40);
}

bool use_lt() {
    const char* e = std::getenv("TCB_OZAKI_LT");  // read per call: tests switch paths in one process
    return e && *e && *e != '0';
}

// out (cols x r, row-major) from the level products: C_L is r_p x cols column-major
__global__ void oz_ttm_combine_kernel(LevelPtrs lv, u64 cols, u64 r, u64 r_p, const int* __restrict__ exc,
                                      const int* __restrict__ exu, double* __restrict__ out) {
    const u64 e = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= cols * r) return;
    const u64 c = e / r, j = e % r;
    const u64 off = c * r_p + j;
    long long T = 0;
#pragma unroll
    for (int L = 0; L < kSlices; ++L) T += static_cast<long long>(lv.c[L][off]) * (1LL << (7 * (kSlices - 1 - L)));
    out[e] = scalbn(static_cast<double>(T), exc[c] + exu[j] - 40);
}

u64 round_up(u64 v, u64 m) { return (v + m - 1) / m * m; }

}  // namespace

bool ozaki_lt_forced() { return use_lt(); }

bool ozaki_gram_ok(u64 rows, u64 cols) {
    const char* e = std::getenv("TCB_OZAKI");  // read per call: tests switch paths in one process
    const bool off = e && *e == '0';
    // cols <= 2^22 keeps the int64 recombination of the Gram levels below 2^63
    return !off && rows >= 256 && cols >= (u64{1} << 18) && cols <= (u64{1} << 22);
}

bool ozaki_ttm_ok(u64 rows, u64 cols, u64 r) {
    return ozaki_gram_ok(rows, cols) && r >= 64 && rows <= 4096;
}

void gram_ozaki(const double* B, u64 rows, u64 cols, double* G, cudaStream_t s) {
    ProfScope prof_scope(kGram, s);
    const u64 rows_p = round_up(rows, 16), Kp = round_up(cols, kGramKC);
    DevBuf<int> ex(rows_p, s);
    DevBuf<double> sq(rows, s);
    ex.zero();
    oz_rowstat_kernel<<<static_cast<unsigned>(rows), 256, 0, s>>>(B, cols, ex.p, sq.p);
    count_launch();
    TCB_LAUNCH();
    if (!use_lt()) {
        const u64 nslab = Kp / kOzSlab;
        const u64 ra = oz_block_rows(rows, kOzBM), rb = oz_block_rows(rows, kOzBN);
        DevBuf<int8_t> da(oz_block_bytes(rows, nslab, kOzBM), s), db(oz_block_bytes(rows, nslab, kOzBN), s);
        oz_split_rows_blk_kernel<<<dim3(cdiv(Kp, 1024), static_cast<unsigned>(std::max(ra, rb))), 256, 0, s>>>(
            B, rows, cols, nslab, ex.p, da.p, ra, db.p, rb, 0);
        count_launch();
        TCB_LAUNCH();
        const u64 ld = oz_gram_acc_ld(rows);
        DevBuf<long long> acc(ra * ld, s);
        acc.zero();
        oz_gram_tc(da.p, db.p, rows, nslab, acc.p, ld, s);
        oz_gram_final_kernel<<<cdiv(rows * rows, 256), 256, 0, s>>>(acc.p, ld, rows, ex.p, sq.p, G);
        count_launch();
        TCB_LAUNCH();
        return;
    }
    const u64 slab = rows_p * kSlices * Kp;
    DevBuf<int8_t> dcat(slab, s), drev(slab, s);
    if (rows_p > rows) {  // zero rows for the padding
        TCB_CUDA(cudaMemsetAsync(dcat.p + rows * kSlices * Kp, 0, (rows_p - rows) * kSlices * Kp, s));
        TCB_CUDA(cudaMemsetAsync(drev.p + rows * kSlices * Kp, 0, (rows_p - rows) * kSlices * Kp, s));
    }
    oz_split_rows_kernel<<<dim3(cdiv(Kp, 1024), static_cast<unsigned>(rows)), 256, 0, s>>>(B, cols, Kp, ex.p, dcat.p,
                                                                                          drev.p);
    count_launch();
    TCB_LAUNCH();
    const u64 mat = rows_p * rows_p;
    const u64 nb_slice = Kp / kGramKC;
    DevBuf<int32_t> part(mat * nb_slice * (kSlices * (kSlices + 1) / 2), s);
    LevelPtrs lv{};
    u64 at = 0;
    for (int L = 0; L < kSlices; ++L) {
        const int nb = static_cast<int>(nb_slice * (L + 1));
        int32_t* c = part.p + at;
        imma_tn(dcat.p, kSlices * Kp, static_cast<long long>(kGramKC), drev.p + (kSlices - 1 - L) * Kp, kSlices * Kp,
                static_cast<long long>(kGramKC), c, rows_p, static_cast<long long>(mat), rows_p, rows_p, kGramKC, nb,
                s);
        count_launch();
        lv.c[L] = c;
        lv.nb[L] = nb;
        at += mat * static_cast<u64>(nb);
    }
    oz_gram_combine_kernel<<<cdiv(rows * rows, 256), 256, 0, s>>>(lv, rows, rows_p, ex.p, sq.p, G);
    count_launch();
    TCB_LAUNCH();
}

// ---- the first Gram while the rows are still arriving (host upload in row slabs)
OzGramRows::OzGramRows(u64 rows_, u64 cols_, cudaStream_t s_) : rows(rows_), cols(cols_), s(s_) {
    nslab = round_up(cols, kGramKC) / kOzSlab;
    ra = oz_block_rows(rows, kOzBM);
    rb = oz_block_rows(rows, kOzBN);
    ld = oz_gram_acc_ld(rows);
    ex = DevBuf<int>(round_up(rows, 16), s);
    ex.zero();
    sq = DevBuf<double>(rows, s);
    da = DevBuf<int8_t>(oz_block_bytes(rows, nslab, kOzBM), s);
    db = DevBuf<int8_t>(oz_block_bytes(rows, nslab, kOzBN), s);
    acc = DevBuf<long long>(ra * ld, s);
    acc.zero();
    const u64 nta = ra / kOzBM, ntb = rb / kOzBN;
    for (u64 a = 0; a < nta; ++a)
        for (u64 b = 0; b < ntb; ++b)
            if (b * kOzBN <= a * kOzBM + kOzBM - 1) pending.push_back(make_int2(static_cast<int>(a), static_cast<int>(b)));
}

void OzGramRows::rows_ready(const double* B, u64 r1) {
    if (r1 <= done || r1 > rows) throw Error("ozaki: rows must arrive in order");
    const u64 r0 = done;
    ProfScope prof_scope(kGram, s);
    oz_rowstat_kernel<<<static_cast<unsigned>(r1 - r0), 256, 0, s>>>(B + r0 * cols, cols, ex.p + r0, sq.p + r0);
    count_launch();
    TCB_LAUNCH();
    // the last slab also writes the zero digits of the padding rows
    const u64 hi = r1 == rows ? std::max(ra, rb) : r1;
    oz_split_rows_blk_kernel<<<dim3(cdiv(nslab * kOzSlab, 1024), static_cast<unsigned>(hi - r0)), 256, 0, s>>>(
        B, rows, cols, nslab, ex.p, da.p, ra, db.p, rb, r0);
    count_launch();
    TCB_LAUNCH();
    done = r1;
    // the tiles whose row blocks are complete now
    std::vector<int2> now, later;
    for (const int2 t : pending) {
        const u64 ea = std::min<u64>(static_cast<u64>(t.x) * kOzBM + kOzBM, rows);
        const u64 eb = std::min<u64>(static_cast<u64>(t.y) * kOzBN + kOzBN, rows);
        (std::max(ea, eb) <= done ? now : later).push_back(t);
    }
    pending.swap(later);
    oz_gram_tc_tiles(da.p, db.p, rows, nslab, now, acc.p, ld, s);
}

void OzGramRows::finish(double* G) {
    if (done != rows || !pending.empty()) throw Error("ozaki: Gram finished before every row arrived");
    oz_gram_final_kernel<<<cdiv(rows * rows, 256), 256, 0, s>>>(acc.p, ld, rows, ex.p, sq.p, G);
    count_launch();
    TCB_LAUNCH();
}

OzTtmPrep::~OzTtmPrep() {
    if (done) cudaEventDestroy(done);
}

std::unique_ptr<OzTtmPrep> ttm_ozaki_prepare(const double* B, u64 rows, u64 cols, cudaStream_t side) {
    auto p = std::make_unique<OzTtmPrep>();
    p->rows = rows;
    p->cols = cols;
    p->nslab = cdiv(rows, kOzSlab);
    const u64 Kr = p->nslab * kOzSlab, ca = oz_block_rows(cols, kOzBM);
    p->exc = DevBuf<int>(round_up(cols, 16), side);
    p->dt = DevBuf<int8_t>(oz_block_bytes(cols, p->nslab, kOzBM), side);
    oz_colexp_kernel<<<cdiv(cols, 256), 256, 0, side>>>(B, rows, cols, p->exc.p);
    oz_split_cols_blk_kernel<<<dim3(cdiv(ca, 32), cdiv(Kr, kColK)), 256, 0, side>>>(B, rows, cols, ca, p->nslab,
                                                                                   p->exc.p, kOzBM, p->dt.p);
    count_launch(2);
    TCB_LAUNCH();
    TCB_CUDA(cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming));
    TCB_CUDA(cudaEventRecord(p->done, side));
    return p;
}

void ttm_ozaki(const double* B, u64 rows, u64 cols, const double* U, u64 r, double* out, cudaStream_t s,
               OzTtmPrep* prep) {
    ProfScope prof_scope(kTtm, s);
    const bool lt = use_lt();
    const u64 r_p = round_up(r, 16), cols_p = round_up(cols, 16);
    if (!lt && prep && prep->rows == rows && prep->cols == cols) {
        TCB_CUDA(cudaStreamWaitEvent(s, prep->done, 0));
        prep->exc.s = s;  // freed in this stream's order, after the products
        prep->dt.s = s;
        const u64 nslab = prep->nslab, Kr = nslab * kOzSlab, ub = oz_block_rows(r, kOzBN);
        DevBuf<int> exu(r_p, s);
        DevBuf<int8_t> eu(oz_block_bytes(r, nslab, kOzBN), s);
        oz_colexp_kernel<<<cdiv(r, 256), 256, 0, s>>>(U, rows, r, exu.p);
        oz_split_cols_blk_kernel<<<dim3(cdiv(ub, 32), cdiv(Kr, kColK)), 256, 0, s>>>(U, rows, r, ub, nslab,
                                                                                    exu.p, kOzBN, eu.p);
        count_launch(2);
        TCB_LAUNCH();
        oz_ttm_tc(prep->dt.p, cols, eu.p, r, nslab, prep->exc.p, exu.p, out, s);
        return;
    }
    DevBuf<int> exc(cols_p, s), exu(r_p, s);
    oz_colexp_kernel<<<cdiv(cols, 256), 256, 0, s>>>(B, rows, cols, exc.p);
    oz_colexp_kernel<<<cdiv(r, 256), 256, 0, s>>>(U, rows, r, exu.p);
    count_launch(2);
    if (!lt) {
        const u64 nslab = cdiv(rows, kOzSlab), Kr = nslab * kOzSlab;
        const u64 ca = oz_block_rows(cols, kOzBM), ub = oz_block_rows(r, kOzBN);
        DevBuf<int8_t> dt(oz_block_bytes(cols, nslab, kOzBM), s), eu(oz_block_bytes(r, nslab, kOzBN), s);
        oz_split_cols_blk_kernel<<<dim3(cdiv(ca, 32), cdiv(Kr, kColK)), 256, 0, s>>>(B, rows, cols, ca, nslab,
                                                                                    exc.p, kOzBM, dt.p);
        oz_split_cols_blk_kernel<<<dim3(cdiv(ub, 32), cdiv(Kr, kColK)), 256, 0, s>>>(U, rows, r, ub, nslab,
                                                                                    exu.p, kOzBN, eu.p);
        count_launch(2);
        TCB_LAUNCH();
        oz_ttm_tc(dt.p, cols, eu.p, r, nslab, exc.p, exu.p, out, s);
        return;
    }
    const u64 Kr = round_up(rows, 16);
    DevBuf<int8_t> dt(cols_p * kSlices * Kr, s), eu(r_p * kSlices * Kr, s);
    oz_split_cols_kernel<<<dim3(cdiv(cols_p, 32), cdiv(Kr, 32)), 256, 0, s>>>(B, rows, cols, cols_p, Kr, exc.p, 1,
                                                                             dt.p);
    oz_split_cols_kernel<<<dim3(cdiv(r_p, 32), cdiv(Kr, 32)), 256, 0, s>>>(U, rows, r, r_p, Kr, exu.p, 0, eu.p);
    count_launch(2);
    TCB_LAUNCH();
    DevBuf<int32_t> lev(kSlices * r_p * cols_p, s);
    LevelPtrs lv{};
    for (int L = 0; L < kSlices; ++L) {
        int32_t* c = lev.p + static_cast<u64>(L) * r_p * cols_p;
        imma_tn(eu.p, kSlices * Kr, 0, dt.p + (kSlices - 1 - L) * Kr, kSlices * Kr, 0, c, r_p, 0, r_p, cols_p,
                static_cast<u64>(L + 1) * Kr, 1, s);
        count_launch();
        lv.c[L] = c;
        lv.nb[L] = 1;
    }
    oz_ttm_combine_kernel<<<cdiv(cols * r, 256), 256, 0, s>>>(lv, cols, r, r_p, exc.p, exu.p, out);
    count_launch();
    TCB_LAUNCH();
}

}  // namespace tcb
