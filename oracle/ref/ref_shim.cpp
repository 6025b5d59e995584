// TEST INFRASTRUCTURE ONLY.  extern "C" probes over the reference's OWN
// integer translation units (core_codec.cpp, entropy.cpp, error_model.cpp,
// vectorize.cpp, container.cpp, kernels*.cpp compiled verbatim from
// /root/reference/proj/src by oracle/ref/build_ref.sh into oracle/_ref/).
// Used to pin the oracle restatement (oracle/src) bit for bit.
#include <cstdlib>
#include <cstring>
#include <string>

#include "tucomp/container.hpp"
#include "tucomp/core_codec.hpp"
#include "tucomp/entropy.hpp"
#include "tucomp/error_model.hpp"
#include "tucomp/kernels.hpp"
#include "tucomp/vectorize.hpp"

using namespace tucomp;

namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
template <class T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(v.size() * sizeof(T) + 1));
    if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
    return p;
}
void le32(std::vector<uint8_t>& o, uint32_t v) {
    for (int i = 0; i < 4; ++i) o.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void le64(std::vector<uint8_t>& o, uint64_t v) {
    for (int i = 0; i < 8; ++i) o.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
// same layout as the reference's write_stream (container.cpp:231-247)
std::vector<uint8_t> serial(uint64_t count, const corecodec::EncodedCore& e) {
    std::vector<uint8_t> o;
    le64(o, count);
    le64(o, e.block_size);
    o.push_back(static_cast<uint8_t>(e.last_plane));
    le32(o, static_cast<uint32_t>(e.stops.size()));
    for (auto& s : e.stops) {
        le64(o, s.leading);
        le64(o, s.trailing);
    }
    le32(o, static_cast<uint32_t>(e.payloads.size()));
    for (auto& pl : e.payloads)
        for (auto& b : pl) {
            le32(o, static_cast<uint32_t>(b.size()));
            o.insert(o.end(), b.begin(), b.end());
        }
    return o;
}
corecodec::EncodedCore own(const corecodec::CoreMeta& m,
                           const std::vector<std::vector<std::span<const uint8_t>>>& pl) {
    corecodec::EncodedCore e;
    e.last_plane = m.last_plane;
    e.block_size = m.block_size;
    e.stops = m.stops;
    e.payloads.resize(pl.size());
    for (std::size_t i = 0; i < pl.size(); ++i)
        for (auto& b : pl[i]) e.payloads[i].emplace_back(b.begin(), b.end());
    return e;
}
}  // namespace

extern "C" {
const char* ref_last_error(void) { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

int ref_encode(const uint64_t* m, const uint8_t* neg, uint64_t n, double target_int, int coder, uint64_t block,
               int split, int fixed_plane, int workers, uint8_t** out, uint64_t* out_len, int* last_plane,
               double* achieved, uint64_t* decoded) {
    return guard([&] {
        corecodec::EncodeOptions o;
        o.coder = static_cast<entropy::Coder>(coder);
        o.block_size = block;
        o.split_planes = split != 0;
        o.workers = workers;
        if (fixed_plane >= 0) o.fixed_last_plane = fixed_plane;
        corecodec::Encoder enc({m, n}, o);
        enc.plan(target_int);
        if (decoded) std::memcpy(decoded, enc.decoded_magnitudes().data(), n * 8);
        auto e = enc.finalize({neg, n});
        auto b = serial(n, e);
        *out = dup(b);
        *out_len = b.size();
        *last_plane = e.last_plane;
        *achieved = e.achieved_sse_int;
    });
}

int ref_quantize_f64(const double* core, const uint64_t* shape, int d, uint64_t* mag, uint8_t* neg, int* k,
                     int* zero, double* slice_norms) {
    return guard([&] {
        Shape sh(shape, shape + d);
        DenseTensor<double> t(sh, std::vector<double>(core, core + shape_numel(sh)));
        auto om = vectorize::OrderMap::build(vectorize::Method::lexicographic, sh);
        auto q = corecodec::quantize(t, om);
        *k = q.scale_exponent;
        *zero = q.zero_flag;
        if (!q.zero_flag) {
            std::memcpy(mag, q.magnitudes.data(), q.magnitudes.size() * 8);
            std::memcpy(neg, q.signs.data(), q.signs.size());
        }
        std::size_t o = 0;
        for (auto& ax : q.slice_norms)
            for (double s : ax) slice_norms[o++] = s;
    });
}

int ref_order_map(int method, const uint64_t* shape, int d, uint64_t* out) {
    return guard([&] {
        Shape sh(shape, shape + d);
        const auto om = vectorize::OrderMap::build(static_cast<vectorize::Method>(method), sh);
        for (std::uint64_t v = 0; v < om.size(); ++v) out[v] = om[v];
    });
}

// corecodec::quantize with a non-default vectorization (slice norms summed in that order)
int ref_quantize_method_f64(const double* core, const uint64_t* shape, int d, int method, uint64_t* mag,
                            uint8_t* neg, int* k, int* zero, double* slice_norms) {
    return guard([&] {
        Shape sh(shape, shape + d);
        DenseTensor<double> t(sh, std::vector<double>(core, core + shape_numel(sh)));
        auto om = vectorize::OrderMap::build(static_cast<vectorize::Method>(method), sh);
        auto q = corecodec::quantize(t, om);
        *k = q.scale_exponent;
        *zero = q.zero_flag;
        if (!q.zero_flag) {
            std::memcpy(mag, q.magnitudes.data(), q.magnitudes.size() * 8);
            std::memcpy(neg, q.signs.data(), q.signs.size());
        }
        std::size_t o = 0;
        for (auto& ax : q.slice_norms)
            for (double s : ax) slice_norms[o++] = s;
    });
}

int ref_encode_symbols(int coder, const uint64_t* s, uint64_t n, uint8_t** out, uint64_t* len) {
    return guard([&] {
        auto b = entropy::encode_symbols(static_cast<entropy::Coder>(coder), {s, n});
        *out = dup(b);
        *len = b.size();
    });
}

int ref_decode_symbols(const uint8_t* p, uint64_t len, uint64_t** out, uint64_t* n) {
    return guard([&] {
        auto v = entropy::decode_symbols({p, len});
        *out = dup(v);
        *n = v.size();
    });
}

// read_container -> write_container: the verbatim writer re-serialises what
// the verbatim reader parsed; equality with the input pins the oracle's bytes.
int ref_container_rewrite(const uint8_t* c, uint64_t n, uint8_t** out, uint64_t* len) {
    return guard([&] {
        auto p = container::read_container({c, n});
        std::vector<container::FactorPayload> fps;
        for (auto& f : p.factors) {
            container::FactorPayload fp;
            fp.dead = f.dead;
            fp.slice_norms = f.slice_norms;
            fp.scale_exponent = f.scale_exponent;
            fp.coeff_count = f.coeff_count;
            fp.stream = own(f.meta, f.payloads);
            fps.push_back(std::move(fp));
        }
        auto core = own(p.core.meta, p.core.payloads);
        auto b = container::write_container(p.header, fps, core);
        *out = dup(b);
        *len = b.size();
    });
}

// decode every stream of a container with the verbatim decoder; returns the
// core magnitudes/signs (storage order) for comparison.
int ref_container_core(const uint8_t* c, uint64_t n, uint64_t** mag, uint8_t** neg, uint64_t* count) {
    return guard([&] {
        auto p = container::read_container({c, n});
        if (p.header.zero_flag) {
            *count = 0;
            *mag = dup(std::vector<uint64_t>{});
            *neg = dup(std::vector<uint8_t>{});
            return;
        }
        auto d = corecodec::decode(p.core.meta, p.core.payloads, 1);
        *mag = dup(d.magnitudes);
        *neg = dup(d.signs);
        *count = d.magnitudes.size();
    });
}

double ref_sum_squares_f64(const double* x, uint64_t n) { return kernels::sum_squares(x, n); }
double ref_sum_squares_f32(const float* x, uint64_t n) { return kernels::sum_squares(x, n); }
double ref_backward_sum(const uint64_t* m, uint64_t n) { return errormodel::backward_sum_sse(std::span<const uint64_t>(m, n)); }
const char* ref_backend(void) { return kernels::active_backend(); }
}
