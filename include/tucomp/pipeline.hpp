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
}
namespace vectorize {
enum class Method : std::uint8_t { lexicographic = 0, zigzag = 1, zorder = 2 };
}
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

}  // namespace pipeline
}  // namespace tucomp
