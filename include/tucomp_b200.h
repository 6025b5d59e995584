/*
 * tucomp_b200.h — C ABI of the B200 (sm_100a) compress path.
 *
 * Drop-in boundary for the reference operator API
 *   tucomp::pipeline::compress(const container::SourceBuffer&, const Params&)
 *   (/root/reference/proj/include/tucomp/pipeline.hpp:57, implemented at
 *    /root/reference/proj/src/pipeline.cpp:240-252)
 * flattened to plain pointers and sizes so any FFI (ctypes, cgo, JNI, N-API)
 * can bind it; include/tucomp/pipeline.hpp re-exposes it with the reference's
 * C++ types.  Every function returns 0 on success; on failure it returns
 * non-zero and tcb_last_error() holds the reference's error text
 * (e.g. "sthosvd: input contains non-finite values").
 *
 * There is no CPU fallback: every entry point runs CUDA kernels on the
 * current device and fails loudly when no sm_100a device is present.
 */
#ifndef TUCOMP_B200_H
#define TUCOMP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* tucomp::pipeline::Params (pipeline.hpp:14-28), fixed-size arrays for d <= 8 */
typedef struct tcb_params {
    int has_target_re;           /* exactly one of the two targets must be set */
    double target_re;
    int has_target_sse;
    double target_sse;
    double rtmss;                /* errormodel::kDefaultRtmss = 0.5 */
    int threads;                 /* host helper threads (results never depend on it) */
    int method;                  /* vectorize::Method; 0 = lexicographic */
    int has_storage_order;
    uint64_t storage_order[8];
    int has_mode_order;
    uint64_t mode_order[8];
    int coder;                   /* entropy::Coder; 0 = arithmetic, 1 = rANS */
    int split_planes;
    int simple_factor_weights;
    uint64_t block_size;         /* 0 = codec default */
    int internal_float32;
    int svd_backend;             /* sthosvd::SvdBackend; 0 automatic, 1 gram, 2 direct */
} tcb_params;

/* tucomp::pipeline::PhaseTimes (pipeline.hpp:30-37), milliseconds */
typedef struct tcb_times {
    double sthosvd_ms, quantize_ms, core_encode_ms, factor_encode_ms, serialize_ms, total_ms;
} tcb_times;

/* tucomp::pipeline::CompressResult (pipeline.hpp:39-55) */
typedef struct tcb_result {
    uint8_t* container;          /* owned by the library: release with tcb_free */
    uint64_t container_size;
    double truncation_sse, core_quantization_sse, factor_terms[8]; /* ErrorEstimate */
    double estimate_sse;
    double norm_sq, target_sse;
    uint64_t ranks[8];
    int order;
    tcb_times times;
    uint64_t peak_alloc_estimate;
    uint64_t original_bytes;
    int ingest_precision_loss;
    /* device-path diagnostics (no reference counterpart) */
    int core_last_plane, core_scale_exponent;
    int uncertified_decisions;   /* always 0: every encoder decision is made on exact serial sums */
    uint64_t kernel_launches;
    uint32_t rank_tie_modes;     /* bit i: mode i's rank cut lies within the eigenvalue error band of the
                                    budget (another fp64 solver may cut one vector apart) */
} tcb_result;

void tcb_default_params(tcb_params* p);

/* pipeline::compress with a HOST SourceBuffer {bytes, dtype, shape, skip_bytes}
 * (container.hpp:34-39); host->device copy included. dtype = container::Dtype. */
int tcb_compress(const uint8_t* bytes, uint64_t nbytes, int dtype, const uint64_t* shape, int d,
                 uint64_t skip_bytes, const tcb_params* params, tcb_result* out);

/* Same, with the element bytes (after skip) already resident in device memory. */
int tcb_compress_device(const void* device_bytes, uint64_t nbytes, int dtype, const uint64_t* shape, int d,
                        const tcb_params* params, tcb_result* out);

/* Sharded compress over NCCL (SURVEY 8(e), B200 extension): every rank holds an
 * equal slab (local_extent) of the last processed mode, in rank order, of a
 * tensor with the global `shape`; the partial Grams are summed with NCCL, the
 * projections stay local, the small tensor is gathered for the last step and
 * rank 0 writes the container (the other ranks return an empty one).
 * tcb_nccl_unique_id on rank 0, the 128 bytes shared by the caller (e.g.
 * torch.distributed), then tcb_nccl_comm_init on every rank. */
int tcb_nccl_unique_id(uint8_t out[128]);
int tcb_nccl_comm_init(const uint8_t id[128], int world, int rank, void** comm);
int tcb_nccl_comm_destroy(void* comm);
int tcb_compress_sharded_device(void* comm, int world, int rank, const void* device_bytes, uint64_t nbytes,
                                int dtype, const uint64_t* shape, int d, uint64_t local_extent,
                                const tcb_params* params, tcb_result* out);

/* Collectives on host memory supplied by the caller, so the sharded pipeline can
 * run over any transport (e.g. torch.distributed with gloo): in-place fp64 sum
 * and a rank-major all-gather of equal-size byte blocks.  Return 0 on success. */
typedef struct tcb_host_collectives {
    void* ctx;
    int (*allreduce_sum_f64)(void* ctx, double* buf, uint64_t n);
    int (*allgather)(void* ctx, const void* send, void* recv, uint64_t bytes_per_rank);
} tcb_host_collectives;

/* tcb_compress_sharded_device with the collectives above instead of NCCL. */
int tcb_compress_sharded_host(const tcb_host_collectives* coll, int world, int rank, const void* device_bytes,
                              uint64_t nbytes, int dtype, const uint64_t* shape, int d, uint64_t local_extent,
                              const tcb_params* params, tcb_result* out);

/* pipeline::DecompressResult (pipeline.hpp:59-64) */
typedef struct tcb_decompress_result {
    uint8_t* bytes;              /* source-dtype bytes, owned by the library: release with tcb_free */
    uint64_t nbytes;
    int dtype;                   /* container::Dtype of the source */
    int d;
    uint64_t shape[8];
    double total_ms;
} tcb_decompress_result;

/* pipeline::decompress(container_bytes, threads) (pipeline.hpp:66, pipeline.cpp:266-283):
 * decode, reconstruct and emit in the source dtype (container.cpp:98-140). */
int tcb_decompress(const uint8_t* container, uint64_t len, int threads, tcb_decompress_result* out);
/* pipeline::decompress with the emitted source-dtype bytes written to device
 * memory (`device_out`, at least `capacity` bytes; out->bytes is NULL): no
 * host copy of the tensor.  B200 extension of pipeline.hpp:66. */
int tcb_decompress_device(const uint8_t* container, uint64_t len, void* device_out, uint64_t capacity,
                          tcb_decompress_result* out);
/* pipeline::decompress_tensor<double> (pipeline.hpp:70-71): the reconstructed tensor in
 * fp64, row-major, original axis order; *out is released with tcb_free; shape has room for 8. */
int tcb_decompress_tensor_f64(const uint8_t* container, uint64_t len, double** out, uint64_t* count,
                              uint64_t* shape, int* d);

/* The CLI's measure_error (tools/tucomp_main.cpp:121-135): decompress `container`
 * on the device, ingest the source bytes (same meaning as tcb_compress) on the
 * device and return sse_between (tensor.cpp:147-164) of the two; internal_float32
 * compares float-rounded values as the reference's float tensors do. */
int tcb_measure_error(const uint8_t* bytes, uint64_t nbytes, int dtype, const uint64_t* shape, int d, uint64_t skip,
                      int internal_float32, const uint8_t* container, uint64_t len, double* sse);

/* container::Header (container.hpp:59-82) as read by container::read_container
 * (container.cpp:338-420): every header and section-structure check, host only
 * (no device work; the CLI's `info`, tucomp_main.cpp:196-228). Orders are 0-based. */
typedef struct tcb_container_header {
    int version, source_dtype, internal_float32, d, coder, method;
    int zero_flag, split_planes, simple_weights;
    uint64_t mode_sizes[8], ranks[8], processing_order[8], storage_order[8];
    int core_scale_exponent;
    uint64_t block_size;
    double rtmss, target_sse, norm_sq, truncation_sse, core_quant_sse, estimate_sse;
} tcb_container_header;
int tcb_read_container_header(const uint8_t* container, uint64_t len, tcb_container_header* out);

void tcb_free(void* p);
const char* tcb_last_error(void);
uint64_t tcb_kernel_launches(void);
/* Pinned staging buffers (per-thread bounce buffers and upload rings) allocated
 * so far in this process: stops growing once every helper thread has one,
 * since ending threads hand theirs on (a leak check for tests). */
uint64_t tcb_pinned_staging_allocs(void);

/* Per-stage device timing with CUDA events on the launching stream (no
 * reference counterpart; replaces PhaseTimes' wall clocks for roofline work).
 * Stage order: ingest, permute, gram, eig, ttm, quant, stats, emit, ac,
 * factor, sum.  tcb_prof_read synchronizes, returns and clears the totals. */
void tcb_prof_enable(int on);
int tcb_prof_read(double* ms, uint64_t* counts, int nstages);
/* Measured fp64 DMMA throughput of this device (TFLOP/s), the roofline
 * denominator for the Gram/TTM kernels (MEASURED_PEAKS.json has no fp64). */
double tcb_peak_dmma_tflops(void);

/* ---- lower-level entry points on host buffers (each wraps device kernels);
 * the reference symbols they replace are named per function. ---- */

/* sthosvd::compress<double> (sthosvd.hpp:66-68). core: processing order;
 * factors[i]: n_i x r_i row-major; out arrays sized by the caller
 * (core: prod(shape), factors[i]: n_i*n_i). */
int tcb_sthosvd_f64(const double* a, const uint64_t* shape, int d, double sse_target, const uint64_t* order,
                    int backend, double* core, uint64_t* core_shape, double** factors, uint64_t* ranks,
                    double* trunc, uint64_t* order_out);

/* G = B B^T (sthosvd.cpp:78-79), B row-major rows x cols, G full row-major. */
int tcb_gram_f64(const double* b, uint64_t rows, uint64_t cols, double* g);
/* next = B^T U (sthosvd.cpp:158-166), U rows x r row-major, next cols x r. */
int tcb_ttm_f64(const double* b, uint64_t rows, uint64_t cols, const double* u, uint64_t r, double* next);
/* SelfAdjointEigenSolver (sthosvd.cpp:80-90): descending eigenvalues and the
 * top-r eigenvectors (n x r row-major, sign-fixed as sthosvd.cpp:103-110). */
int tcb_eig_f64(const double* g, uint64_t n, uint64_t r, double* evals_desc, double* u);

/* corecodec::quantize (core_codec.cpp:55-93), lexicographic order. */
int tcb_quantize_f64(const double* core, const uint64_t* shape, int d, uint64_t* mag, uint8_t* neg, int* k,
                     int* zero, double* slice_norms);

/* corecodec::Encoder plan+finalize (core_codec.cpp:173-413); *stream receives
 * the serialized stream section (container.cpp:231-247). fixed_plane < 0: none. */
int tcb_encode(const uint64_t* mag, const uint8_t* neg, uint64_t n, double target_sse_int, int coder,
               uint64_t block_size, int split, int fixed_plane, uint8_t** stream, uint64_t* stream_len,
               int* last_plane, double* achieved_sse_int, uint64_t* decoded, int* uncertified);

/* The encoder's serial double sums, bit-exact (exact.cu): for every kind k and
 * segment g, s = seg_s0[g]; for each element of [seg_lo, seg_hi) (descending
 * when seg_backward) s = fl(s + term_k(element)); with a finite seg_need the
 * scan stops after the first element that brings s to >= need (place_stops).
 * Terms (kind_term): 0 lead gain, 1 trail gain, 2 both (non-split scan) at
 * kind_plane -- build_block's statistics, core_codec.cpp:131-155, 268-341;
 * 3 (double)m^2 -- backward_sum_sse, error_model.cpp:34-41; 4 recalibrate_sse's
 * term, error_model.cpp:54-72; 5 (m - dec)^2 -- core_codec.cpp:405-411.
 * Outputs indexed k * nseg + g; c0 / c1 count lead / trail positions (lead
 * kind: c1 = new ones) up to the crossing.  reference != 0: the plain
 * one-thread serial chain (verification). */
int tcb_exact_sums(const uint64_t* mag, const uint64_t* dec, uint64_t n, const uint64_t* seg_lo,
                   const uint64_t* seg_hi, const int* seg_backward, const double* seg_s0, const double* seg_need,
                   int nseg, const int* kind_term, const int* kind_plane, int nk, int reference, double* sums,
                   uint64_t* c0, uint64_t* c1, int* crossed);

/* build_block's per-block statistics (core_codec.cpp:131-155) of planes
 * p_top .. p_top-np+1 (np <= 32) over blocks of block_size elements, bit-exact:
 * outputs indexed (2 (p_top - p) + {0 lead, 1 trail}) * nblocks + b, as
 * tcb_exact_sums returns them for those kinds. */
int tcb_exact_plane_stats(const uint64_t* mag, uint64_t n, uint64_t block_size, int p_top, int np, double* sums,
                          uint64_t* c0, uint64_t* c1, int* crossed);

/* entropy::encode_symbols (entropy.cpp:429-445) for one symbol sequence. */
int tcb_encode_symbols(int coder, const uint64_t* syms, uint64_t n, uint8_t** out, uint64_t* len);

/* factorcodec::encode_factor<double> (factor_codec.cpp:153-244). */
int tcb_encode_factor_f64(const double* u, uint64_t n, uint64_t r, const uint8_t* dead, const double* slice_norms,
                          int coder, int simple, int core_step_log2, double term_cap, uint8_t** stream,
                          uint64_t* len, int* k, uint64_t* count, int8_t* flips, double* term, int* plane);

/* ---- device-pointer building blocks of the sharded multi-GPU mode loop
 * (paper_2107_01384_b200/shard.py).  All pointers are device
 * pointers on the current device; capacities as noted. ---- */

/* ||x||^2 and the all-finite flag (tensor.cpp:152-155, sthosvd.cpp:118). */
int tcb_dev_sumsq(const double* x, uint64_t n, double* out, int* finite);
/* row-major axis permutation (tensor.cpp:105-144). */
int tcb_dev_permute(const double* src, double* dst, const uint64_t* shape, const uint64_t* perm, int d);
/* partial Gram of a column shard: g (rows x rows) = b b^T (sthosvd.cpp:79). */
int tcb_dev_gram(const double* b, uint64_t rows, uint64_t cols, double* g);
/* eigensolve + rank rule + sign fix of an all-reduced Gram (sthosvd.cpp:80-90,144-156);
 * u capacity n*n, receives n x r row-major. */
int tcb_dev_factor_from_gram(const double* g, uint64_t n, double budget, double* u, uint64_t* r, double* discarded);
/* one replicated mode step (sthosvd.cpp:136-166); u cap rows*rows, next cap cols*rows. */
int tcb_dev_mode_step(const double* b, uint64_t rows, uint64_t cols, double budget, int backend, double* u,
                      double* next, uint64_t* r, double* discarded);
/* shard-local projection next (cols x r) = b^T u (sthosvd.cpp:158-166). */
int tcb_dev_ttm(const double* b, uint64_t rows, uint64_t cols, const double* u, uint64_t r, double* next);
/* the same Gram / projection by the Ozaki scheme on the INT8 tensor cores (five
 * digit slices per row / column, exact integer recombination; what the mode loop
 * uses for large unfoldings); any rows / cols / r. */
int tcb_dev_gram_ozaki(const double* b, uint64_t rows, uint64_t cols, double* g);
int tcb_dev_ttm_ozaki(const double* b, uint64_t rows, uint64_t cols, const double* u, uint64_t r, double* next);
/* phases 2-5 of compress_impl (pipeline.cpp:77-189) on a device factorization
 * (core in processing order, factors[i] n_i x r_i row-major). */
int tcb_dev_encode_tucker(const double* core, const double* const* factors, const uint64_t* n, const uint64_t* r,
                          const uint64_t* order, const double* trunc, int d, int dtype, double norm_sq,
                          double target_sse, const tcb_params* params, tcb_result* out);
/* The same encode split over `world` ranks (each rank holds the whole Tucker and
 * codes its share of the core's blocks); coll == NULL with
 * nccl_comm != NULL uses NCCL.  Rank 0's container equals the unsharded one. */
int tcb_dev_encode_tucker_sharded(void* nccl_comm, const tcb_host_collectives* coll, int world, int rank,
                                  const double* core, const double* const* factors, const uint64_t* n,
                                  const uint64_t* r, const uint64_t* order, const double* trunc, int d, int dtype,
                                  double norm_sq, double target_sse, const tcb_params* params, tcb_result* out);

#ifdef __cplusplus
}
#endif

#endif /* TUCOMP_B200_H */
