// Drop-in C++ surface for the reference's compress API on the B200 path.
//
// Mirrors /root/reference/proj/include/tucomp/pipeline.hpp:14-71 (Params,
// PhaseTimes, CompressResult, compress) and the container/errormodel types it
// uses (container.hpp:16-39, error_model.hpp:36-46, tensor.hpp:14-17), with
// no Eigen types (the reference's Matrix<T> alias is not part of this
// surface).  Header-only: every call forwards to the C ABI in
// include/tucomp_b200.h (libtucomp_b200.so, sm_100a kernels); errors are
// rethrown as tucomp::Error with the reference's message text.
#pragma once

#include <cstdint>
#include <cstring>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../tucomp_b200.h"

namespace tucomp {

class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

using Shape = std::vector<std::size_t>;
using ModePermutation = std::vector<std::size_t>;

namespace container {
enum class Dtype : std::uint8_t { int8 = 0, uint8, int16, uint16, int32, uint32, int64, uint64, float32, float64 };
struct SourceBuffer {
    std::span<const std::uint8_t> bytes;
    Dtype dtype = Dtype::float64;
    Shape shape;
    std::size_t skip_bytes = 0;
};
}  // namespace container

namespace entropy {
enum class Coder : std::uint8_t { arithmetic = 0, rans = 1 };
// entropy.cpp:10-19
inline const char* coder_name(Coder c) { return c == Coder::arithmetic ? "ac" : "rans"; }
inline std::optional<Coder> coder_from_name(const std::string& s) {
    if (s == "ac" || s == "arithmetic") return Coder::arithmetic;
    if (s == "rans") return Coder::rans;
    return std::nullopt;
}
}  // namespace entropy
namespace vectorize {
enum class Method : std::uint8_t { lexicographic = 0, zigzag = 1, zorder = 2 };
// vectorize.cpp:9-22
inline const char* method_name(Method m) {
    static const char* const names[] = {"lex", "zigzag", "zorder"};
    return static_cast<unsigned>(m) < 3 ? names[static_cast<unsigned>(m)] : "?";
}
inline std::optional<Method> method_from_name(const std::string& s) {
    if (s == "lex" || s == "lexicographic") return Method::lexicographic;
    if (s == "zigzag") return Method::zigzag;
    if (s == "zorder") return Method::zorder;
    return std::nullopt;
}
}  // namespace vectorize

namespace container {
inline constexpr std::uint8_t kFormatVersion = 1;
// container.cpp:9-47
inline const char* dtype_name(Dtype t) {
    static const char* const names[] = {"int8",  "uint8",  "int16",  "uint16",  "int32",
                                        "uint32", "int64", "uint64", "float32", "float64"};
    return static_cast<unsigned>(t) < 10 ? names[static_cast<unsigned>(t)] : "?";
}
inline std::size_t dtype_size(Dtype t) {
    static const std::size_t sizes[] = {1, 1, 2, 2, 4, 4, 8, 8, 4, 8};
    return static_cast<unsigned>(t) < 10 ? sizes[static_cast<unsigned>(t)] : 0;
}
inline std::optional<Dtype> dtype_from_name(const std::string& s) {
    for (unsigned i = 0; i < 10; ++i)
        if (s == dtype_name(static_cast<Dtype>(i))) return static_cast<Dtype>(i);
    return std::nullopt;
}

// container.hpp:59-82 (orders 0-based)
struct Header {
    Dtype source_dtype = Dtype::float64;
    bool internal_float32 = false;
    std::vector<std::uint64_t> mode_sizes, ranks;
    ModePermutation processing_order, storage_order;
    vectorize::Method method = vectorize::Method::lexicographic;
    entropy::Coder coder = entropy::Coder::arithmetic;
    bool zero_flag = false, split_planes = true, simple_weights = false;
    std::int32_t core_scale_exponent = 0;
    std::uint64_t block_size = 0;
    double rtmss = 0.5, target_sse = 0, norm_sq = 0, truncation_sse = 0, core_quant_sse = 0, estimate_sse = 0;

    std::size_t order() const { return mode_sizes.size(); }
    std::uint64_t element_count() const {
        std::uint64_t n = 1;
        for (auto v : mode_sizes) n *= v;
        return n;
    }
};
struct ParsedContainer {  // the header part of container.hpp's ParsedContainer
    Header header;
};

// container::read_container (container.cpp:338-420): header plus the structural
// checks of every section; host only.
inline ParsedContainer read_container(std::span<const std::uint8_t> bytes) {
    tcb_container_header c;
    if (tcb_read_container_header(bytes.data(), bytes.size(), &c) != 0) throw Error(tcb_last_error());
    ParsedContainer p;
    Header& h = p.header;
    h.source_dtype = static_cast<Dtype>(c.source_dtype);
    h.internal_float32 = c.internal_float32 != 0;
    for (int i = 0; i < c.d; ++i) {
        h.mode_sizes.push_back(c.mode_sizes[i]);
        h.ranks.push_back(c.ranks[i]);
        h.processing_order.push_back(c.processing_order[i]);
        h.storage_order.push_back(c.storage_order[i]);
    }
    h.method = static_cast<vectorize::Method>(c.method);
    h.coder = static_cast<entropy::Coder>(c.coder);
    h.zero_flag = c.zero_flag != 0;
    h.split_planes = c.split_planes != 0;
    h.simple_weights = c.simple_weights != 0;
    h.core_scale_exponent = c.core_scale_exponent;
    h.block_size = c.block_size;
    h.rtmss = c.rtmss;
    h.target_sse = c.target_sse;
    h.norm_sq = c.norm_sq;
    h.truncation_sse = c.truncation_sse;
    h.core_quant_sse = c.core_quant_sse;
    h.estimate_sse = c.estimate_sse;
    return p;
}
}  // namespace container
namespace sthosvd {
enum class SvdBackend { automatic, gram, direct };
}

namespace errormodel {
inline constexpr double kDefaultRtmss = 0.5;
struct ErrorEstimate {
    double truncation_sse = 0.0;
    double core_quantization_sse = 0.0;
    std::vector<double> factor_terms;
    double total() const {
        double t = truncation_sse + core_quantization_sse;
        for (double f : factor_terms) t += f;
        return t;
    }
};
}  // namespace errormodel

namespace pipeline {

struct Params {
    std::optional<double> target_re;
    std::optional<double> target_sse;
    double rtmss = errormodel::kDefaultRtmss;
    int threads = 1;
    vectorize::Method method = vectorize::Method::lexicographic;
    std::optional<ModePermutation> storage_order;
    std::optional<ModePermutation> mode_order;
    entropy::Coder coder = entropy::Coder::arithmetic;
    bool split_planes = true;
    bool simple_factor_weights = false;
    std::uint64_t block_size = 0;
    bool internal_float32 = false;
    sthosvd::SvdBackend svd_backend = sthosvd::SvdBackend::automatic;
};

struct PhaseTimes {
    double sthosvd_ms = 0, quantize_ms = 0, core_encode_ms = 0, factor_encode_ms = 0, serialize_ms = 0,
           total_ms = 0;
};

struct CompressResult {
    std::vector<std::uint8_t> container;
    errormodel::ErrorEstimate estimate;
    double norm_sq = 0;
    double target_sse = 0;
    std::vector<std::uint64_t> ranks;
    PhaseTimes times;
    std::uint64_t peak_alloc_estimate = 0;
    std::uint64_t original_bytes = 0;
    bool ingest_precision_loss = false;

    double compression_factor() const {
        return container.empty() ? 0.0
                                 : static_cast<double>(original_bytes) / static_cast<double>(container.size());
    }
};

namespace detail {
inline tcb_params to_c(const Params& p, std::size_t d) {
    tcb_params c;
    tcb_default_params(&c);
    c.has_target_re = p.target_re.has_value();
    c.target_re = p.target_re.value_or(0.0);
    c.has_target_sse = p.target_sse.has_value();
    c.target_sse = p.target_sse.value_or(0.0);
    c.rtmss = p.rtmss;
    c.threads = p.threads;
    c.method = static_cast<int>(p.method);
    if (p.storage_order) {
        c.has_storage_order = 1;
        for (std::size_t i = 0; i < d && i < 8; ++i) c.storage_order[i] = (*p.storage_order)[i];
    }
    if (p.mode_order) {
        c.has_mode_order = 1;
        for (std::size_t i = 0; i < d && i < 8; ++i) c.mode_order[i] = (*p.mode_order)[i];
    }
    c.coder = static_cast<int>(p.coder);
    c.split_planes = p.split_planes;
    c.simple_factor_weights = p.simple_factor_weights;
    c.block_size = p.block_size;
    c.internal_float32 = p.internal_float32;
    c.svd_backend = static_cast<int>(p.svd_backend);
    return c;
}
inline CompressResult from_c(tcb_result& r) {
    CompressResult o;
    o.container.assign(r.container, r.container + r.container_size);
    tcb_free(r.container);
    o.estimate.truncation_sse = r.truncation_sse;
    o.estimate.core_quantization_sse = r.core_quantization_sse;
    o.estimate.factor_terms.assign(r.factor_terms, r.factor_terms + r.order);
    o.norm_sq = r.norm_sq;
    o.target_sse = r.target_sse;
    o.ranks.assign(r.ranks, r.ranks + r.order);
    o.times = {r.times.sthosvd_ms,       r.times.quantize_ms,  r.times.core_encode_ms,
               r.times.factor_encode_ms, r.times.serialize_ms, r.times.total_ms};
    o.peak_alloc_estimate = r.peak_alloc_estimate;
    o.original_bytes = r.original_bytes;
    o.ingest_precision_loss = r.ingest_precision_loss != 0;
    return o;
}
}  // namespace detail

// pipeline::compress (reference pipeline.cpp:240-252) on the B200.
inline CompressResult compress(const container::SourceBuffer& src, const Params& params) {
    std::vector<std::uint64_t> shape(src.shape.begin(), src.shape.end());
    const tcb_params c = detail::to_c(params, shape.size());
    tcb_result r;
    if (tcb_compress(src.bytes.data(), src.bytes.size(), static_cast<int>(src.dtype), shape.data(),
                     static_cast<int>(shape.size()), src.skip_bytes, &c, &r) != 0)
        throw Error(tcb_last_error());
    return detail::from_c(r);
}

struct DecompressResult {  // reference pipeline.hpp:59-64
    std::vector<std::uint8_t> bytes;
    container::Dtype dtype = container::Dtype::float64;
    Shape shape;
    double total_ms = 0;
};

// pipeline::decompress (reference pipeline.cpp:266-283) on the B200.
inline DecompressResult decompress(std::span<const std::uint8_t> container_bytes, int threads) {
    tcb_decompress_result r;
    if (tcb_decompress(container_bytes.data(), container_bytes.size(), threads, &r) != 0)
        throw Error(tcb_last_error());
    DecompressResult o;
    o.bytes.assign(r.bytes, r.bytes + r.nbytes);
    tcb_free(r.bytes);
    o.dtype = static_cast<container::Dtype>(r.dtype);
    o.shape.assign(r.shape, r.shape + r.d);
    o.total_ms = r.total_ms;
    return o;
}

// pipeline::decompress_tensor<T> (pipeline.hpp:70-71): the reconstruction in the
// original axis order, row-major.  The device computes in fp64; T = float rounds.
template <class T>
inline std::vector<T> decompress_tensor(std::span<const std::uint8_t> container_bytes, int threads = 1) {
    (void)threads;
    double* p = nullptr;
    std::uint64_t n = 0, shape[8];
    int d = 0;
    if (tcb_decompress_tensor_f64(container_bytes.data(), container_bytes.size(), &p, &n, shape, &d) != 0)
        throw Error(tcb_last_error());
    std::vector<T> out(p, p + n);
    tcb_free(p);
    return out;
}

// B200 extension: the CLI's measure_error (tucomp_main.cpp:121-135) with the
// ingest, decompress and SSE on the device; returns the SSE.
inline double measure_sse(const container::SourceBuffer& src, std::span<const std::uint8_t> container_bytes,
                          bool internal_float32) {
    std::vector<std::uint64_t> shape(src.shape.begin(), src.shape.end());
    double sse = 0;
    if (tcb_measure_error(src.bytes.data(), src.bytes.size(), static_cast<int>(src.dtype), shape.data(),
                          static_cast<int>(shape.size()), src.skip_bytes, internal_float32 ? 1 : 0,
                          container_bytes.data(), container_bytes.size(), &sse) != 0)
        throw Error(tcb_last_error());
    return sse;
}

}  // namespace pipeline
}  // namespace tucomp
