// CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain C++ restatement of the reference compress path (ATC / `tucomp`,
// /root/reference/proj) used as the parity checker for the B200 build.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it.  It is never part of the product path.
//
// Integer/bitstream parts (entropy, core codec, container) restate the
// reference bit for bit and are pinned against the reference's own sources
// compiled verbatim into oracle/_ref (see oracle/ref/build_ref.sh).
// Floating-point parts (Gram, eigensolver, SVD, TTM, Householder) restate the
// algorithms Eigen implements; Eigen is absent from this machine, so those are
// "parity unpinned" against Eigen and pinned against numpy/LAPACK instead.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

using u8 = std::uint8_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;
using Shape = std::vector<std::size_t>;
using Perm = std::vector<std::size_t>;
using Bytes = std::vector<u8>;

inline constexpr u64 kFull = ~u64{0};  // "whole block" stop sentinel (core_codec.cpp:14)

// ---------------------------------------------------------------- tensor helpers
std::size_t numel(const Shape& s);
std::vector<std::size_t> strides_of(const Shape& s);  // row-major, last fastest
bool valid_perm(const Perm& p);
Perm inverse_perm(const Perm& p);
Perm stable_ascending(const Shape& s);  // sthosvd.cpp:28-33, vectorize.cpp:25-30
template <class T>
std::vector<T> permute_axes(const std::vector<T>& src, const Shape& shape, const Perm& p);

// ---------------------------------------------------------------- reductions (kernels*.cpp)
double sum_sq(const double* x, std::size_t n);  // AVX2 accumulation order, kernels_avx2.cpp:132-141
double sum_sq(const float* x, std::size_t n);   // kernels_avx2.cpp:143-156
double max_abs_d(const double* x, std::size_t n);
float max_abs_f(const float* x, std::size_t n);
template <class T>
bool finite_all(const T* x, std::size_t n);

// ---------------------------------------------------------------- entropy (entropy.cpp)
enum class Coder : u8 { ac = 0, rans = 1 };

class BitSink {  // MSB-first (entropy.cpp:22-33)
public:
    void put(bool b);
    std::size_t bits() const { return nbits_; }
    Bytes& bytes() { return buf_; }

private:
    Bytes buf_;
    std::size_t nbits_ = 0;
};

std::vector<u64> zero_runs(const std::vector<u8>& column);  // entropy.cpp:51-64
Bytes pack_symbols(Coder c, std::span<const u64> syms);       // entropy.cpp:429-445
std::vector<u64> unpack_symbols(std::span<const u8> payload); // entropy.cpp:447-468

// ---------------------------------------------------------------- core codec (core_codec.cpp)
struct Quantized {
    std::vector<u64> mag;
    std::vector<u8> neg;
    int k = 0;
    bool zero = false;
    Shape shape;
    std::vector<std::vector<double>> slice_norms;
};
template <class T>
Quantized quantize(const std::vector<T>& core, const Shape& shape, std::span<const u64> order = {});
// vectorize::OrderMap (vectorize.cpp:40-170): flat position of the v-th coefficient;
// empty = lexicographic (identity).  method: 0 lexicographic, 1 zigzag, 2 zorder
std::vector<u64> order_map(int method, const Shape& shape);

struct Stops {
    u64 lead = 0, trail = 0;
};

struct Stream {  // EncodedCore (core_codec.hpp:36-45)
    int last_plane = 63;
    u64 block = 0;
    std::vector<Stops> stops;
    std::vector<std::vector<Bytes>> payloads;  // [63 - plane][block]
    double achieved_int = 0.0;
    u64 payload_bytes() const;
};

struct CodecOpts {
    Coder coder = Coder::ac;
    u64 block = 0;
    bool split = true;
    std::optional<int> fixed_plane;
};

u64 default_block(u64 n);

// Encoder planning state exposed for parity probes.
struct Plan {
    int last_plane = 63;
    std::vector<Stops> stops;
    std::vector<u64> decoded;
    std::vector<std::pair<int, double>> trace;
    int n_planes = 0;  // number of stored planes (63 - last_plane + 1, or 0)
};

class CoreEncoder {
public:
    CoreEncoder(std::span<const u64> m, const CodecOpts& o);
    void plan(double target_int);
    Stream finalize(std::span<const u8> neg);
    const Plan& planned() const { return plan_; }

private:
    struct Tally {
        double red_lead = 0, red_trail = 0;
        u64 lead = 0, ones = 0, trail = 0, ebits = 0;
    };
    Bytes emit(int p, std::size_t b, u64 lead_stop, u64 trail_stop, const u8* neg, Tally* t) const;
    void stops_at(int p, double need, const Tally& tot, const std::vector<Tally>& per, const Tally* prev);
    void decode_model();
    std::size_t lo_of(std::size_t b) const { return b * bs_; }
    std::size_t hi_of(std::size_t b) const;

    std::span<const u64> m_;
    CodecOpts o_;
    u64 bs_ = 0;
    std::size_t nb_ = 0;
    std::vector<signed char> top_;
    Plan plan_;
    bool done_ = false;
};

struct StreamMeta {
    u64 count = 0, block = 0;
    int last_plane = 63;
    std::vector<Stops> stops;
};
struct Decoded {
    std::vector<u64> mag;
    std::vector<u8> neg;
};
Decoded decode_stream(const StreamMeta& meta, const std::vector<std::vector<std::span<const u8>>>& pl);
std::vector<std::vector<u8>> dead_slices(const Shape& shape, std::span<const u64> decoded,
                                         std::span<const u64> order = {});

// ---------------------------------------------------------------- error model (error_model.cpp)
double backward_sq(std::span<const u64> v);
double backward_sq(std::span<const double> v);
bool recal_due(u64 terms, double ref, double running);
double recal_sse(std::span<const u64> m, int plane);

// ---------------------------------------------------------------- linear algebra (Eigen stand-ins)
// Column-major n x n symmetric eigen-decomposition (lower triangle read);
// eigenvalues ascending, vectors in columns — SelfAdjointEigenSolver semantics.
template <class T>
void sym_eig(std::vector<T>& a, std::size_t n, std::vector<T>& evals);
// Thin SVD of a row-major rows x cols matrix with rows > cols (BDCSVD stand-in):
// u is column-major rows x cols, sv descending.
template <class T>
void thin_svd(const T* b, std::size_t rows, std::size_t cols, std::vector<T>& u, std::vector<T>& sv);

// ---------------------------------------------------------------- sthosvd (sthosvd.cpp)
enum class SvdBackend { automatic = 0, gram = 1, direct = 2 };
struct RankChoice {
    std::size_t r;
    double discarded;
};
RankChoice pick_rank(std::span<const double> s2, double budget);  // sthosvd.cpp:13-26

template <class T>
struct Tucker {
    std::vector<T> core;  // processing order
    Shape core_shape;
    std::vector<std::vector<T>> factors;  // row-major n_i x r_i, by original mode
    std::vector<std::size_t> n, r;
    Perm order;
    std::vector<double> trunc;                 // by original mode
    std::vector<std::vector<double>> sigma2;   // per step, descending
};
template <class T>
Tucker<T> sthosvd(const std::vector<T>& a, const Shape& shape, double target,
                  const std::optional<Perm>& order, SvdBackend be);
template <class T>
std::vector<T> tucker_expand(const Tucker<T>& f);  // sthosvd.cpp:173-218 (any order; plain)

// ---------------------------------------------------------------- factor codec (factor_codec.cpp)
template <class T>
struct FactorOut {
    std::vector<u8> dead;
    int k = 0;
    u64 count = 0;
    Stream stream;
    std::vector<signed char> flips;
    std::vector<T> decoded;  // row-major n x r
    double term = 0.0;
    int plane = 0;
};
struct FactorOpts {
    Coder coder = Coder::ac;
    bool simple = false;
    int core_step_log2 = 0;
    double term_cap = 0.0;
};
std::vector<double> alpha_weights(std::span<const double> sn, std::size_t n);
template <class T>
FactorOut<T> encode_factor(const std::vector<T>& u, std::size_t n, std::size_t r,
                           std::span<const u8> dead, std::span<const double> sn, const FactorOpts& o);
template <class T>
std::vector<T> decode_factor(std::size_t n, std::size_t r, std::span<const u8> dead,
                             std::span<const double> sn, bool simple, int k, u64 count,
                             const StreamMeta& meta,
                             const std::vector<std::vector<std::span<const u8>>>& pl);

// ---------------------------------------------------------------- container + pipeline
enum class Dtype : u8 { i8 = 0, u8_ = 1, i16 = 2, u16 = 3, i32 = 4, u32_ = 5, i64 = 6, u64_ = 7, f32 = 8, f64 = 9 };
std::size_t dtype_bytes(Dtype t);

struct Params {
    std::optional<double> target_re, target_sse;
    double rtmss = 0.5;
    std::optional<Perm> storage_order, mode_order;
    Coder coder = Coder::ac;
    bool split = true;
    bool simple = false;
    u64 block = 0;
    bool f32 = false;
    SvdBackend backend = SvdBackend::automatic;
    int method = 0;  // vectorize::Method
};

struct Result {
    Bytes container;
    double norm_sq = 0, target_sse = 0;
    double trunc = 0, core_quant = 0, estimate = 0;
    std::vector<double> factor_terms;
    std::vector<u64> ranks;
    u64 original_bytes = 0;
    bool precision_loss = false;
    int core_last_plane = 63;
    int core_k = 0;
    // timing of the phases (ms), PhaseTimes semantics (pipeline.hpp:30-37)
    double t_sthosvd = 0, t_quant = 0, t_core = 0, t_factor = 0, t_ser = 0, t_total = 0;
};

Result compress(std::span<const u8> bytes, Dtype dt, const Shape& shape, std::size_t skip,
                const Params& p);
template <class T>
std::vector<T> decompress_tensor(std::span<const u8> cont, Shape& shape_out);

}  // namespace orc
