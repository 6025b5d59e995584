// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp).
// extern "C" surface loaded by tests/ (ctypes) and bench.py's CPU baseline.
#include <cstdlib>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <cstring>
#include <string>

#include "orc.hpp"

using namespace orc;

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

Shape to_shape(const uint64_t* s, int d) { return Shape(s, s + d); }

// serialized stream section exactly as container.cpp:231-247 writes it
Bytes serial(u64 count, const Stream& s) {
    Bytes o;
    auto u32v = [&](u32 v) {
        for (int i = 0; i < 4; ++i) o.push_back(static_cast<u8>(v >> (8 * i)));
    };
    auto u64v = [&](u64 v) {
        for (int i = 0; i < 8; ++i) o.push_back(static_cast<u8>(v >> (8 * i)));
    };
    u64v(count);
    u64v(s.block);
    o.push_back(static_cast<u8>(s.last_plane));
    u32v(static_cast<u32>(s.stops.size()));
    for (auto& st : s.stops) {
        u64v(st.lead);
        u64v(st.trail);
    }
    u32v(static_cast<u32>(s.payloads.size()));
    for (auto& pl : s.payloads)
        for (auto& b : pl) {
            u32v(static_cast<u32>(b.size()));
            o.insert(o.end(), b.begin(), b.end());
        }
    return o;
}
}  // namespace

extern "C" {

// host threads the oracle's Gram / projection loops use (OpenMP; results do
// not depend on it)
int orc_order_map(int method, const uint64_t* shape, int d, uint64_t* out) {
    return guard([&] {
        const Shape sh(shape, shape + d);
        const auto o = order_map(method, sh);
        const u64 n = numel(sh);
        for (u64 v = 0; v < n; ++v) out[v] = o.empty() ? v : o[v];
    });
}

int orc_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

struct orc_params {
    int has_re;
    double re;
    int has_sse;
    double sse;
    double rtmss;
    int coder;
    int split;
    int simple;
    int f32;
    int backend;
    uint64_t block;
    int has_storage;
    uint64_t storage[8];
    int has_mode;
    uint64_t mode[8];
    int method;  // vectorize::Method
};

struct orc_result {
    uint8_t* container;
    uint64_t size;
    double norm_sq, target_sse, trunc, core_quant, estimate;
    double factor_terms[8];
    uint64_t ranks[8];
    int d;
    int core_last_plane;
    int core_k;
    int precision_loss;
    uint64_t original_bytes;
    double t_sthosvd, t_quant, t_core, t_factor, t_ser, t_total;
};

const char* orc_last_error(void) { return g_err.c_str(); }
void orc_free(void* p) { std::free(p); }

int orc_compress(const uint8_t* bytes, uint64_t n, int dtype, const uint64_t* shape, int d, uint64_t skip,
                 const orc_params* pp, orc_result* out) {
    return guard([&] {
        Params p;
        if (pp->has_re) p.target_re = pp->re;
        if (pp->has_sse) p.target_sse = pp->sse;
        p.rtmss = pp->rtmss;
        p.coder = static_cast<Coder>(pp->coder);
        p.split = pp->split != 0;
        p.simple = pp->simple != 0;
        p.f32 = pp->f32 != 0;
        p.backend = static_cast<SvdBackend>(pp->backend);
        p.method = pp->method;
        p.block = pp->block;
        if (pp->has_storage) p.storage_order = Perm(pp->storage, pp->storage + d);
        if (pp->has_mode) p.mode_order = Perm(pp->mode, pp->mode + d);
        Result r = compress({bytes, n}, static_cast<Dtype>(dtype), to_shape(shape, d), skip, p);
        out->container = dup(r.container);
        out->size = r.container.size();
        out->norm_sq = r.norm_sq;
        out->target_sse = r.target_sse;
        out->trunc = r.trunc;
        out->core_quant = r.core_quant;
        out->estimate = r.estimate;
        for (int i = 0; i < d && i < 8; ++i) {
            out->factor_terms[i] = i < static_cast<int>(r.factor_terms.size()) ? r.factor_terms[i] : 0.0;
            out->ranks[i] = r.ranks[i];
        }
        out->d = d;
        out->core_last_plane = r.core_last_plane;
        out->core_k = r.core_k;
        out->precision_loss = r.precision_loss;
        out->original_bytes = r.original_bytes;
        out->t_sthosvd = r.t_sthosvd;
        out->t_quant = r.t_quant;
        out->t_core = r.t_core;
        out->t_factor = r.t_factor;
        out->t_ser = r.t_ser;
        out->t_total = r.t_total;
    });
}

int orc_decompress_f64(const uint8_t* c, uint64_t n, double** out, uint64_t* len) {
    return guard([&] {
        Shape s;
        auto v = decompress_tensor<double>({c, n}, s);
        *out = dup(v);
        *len = v.size();
    });
}

int orc_decompress_f32(const uint8_t* c, uint64_t n, float** out, uint64_t* len) {
    return guard([&] {
        Shape s;
        auto v = decompress_tensor<float>({c, n}, s);
        *out = dup(v);
        *len = v.size();
    });
}

// ST-HOSVD probe: core (processing order) and per-mode factors (row-major n_i x r_i)
int orc_sthosvd_f64(const double* a, const uint64_t* shape, int d, double target, const uint64_t* order,
                    int backend, double** core, uint64_t* core_shape, double** factors, uint64_t* ranks,
                    double* trunc, double** sigma2, uint64_t* sigma2_len, uint64_t* order_out) {
    return guard([&] {
        const Shape sh = to_shape(shape, d);
        std::vector<double> x(a, a + numel(sh));
        std::optional<Perm> ord;
        if (order) ord = Perm(order, order + d);
        auto f = sthosvd(x, sh, target, ord, static_cast<SvdBackend>(backend));
        *core = dup(f.core);
        for (int i = 0; i < d; ++i) {
            core_shape[i] = f.core_shape[i];
            factors[i] = dup(f.factors[i]);
            ranks[i] = f.r[i];
            trunc[i] = f.trunc[i];
            sigma2[i] = dup(f.sigma2[i]);
            sigma2_len[i] = f.sigma2[i].size();
            order_out[i] = f.order[i];
        }
    });
}

int orc_eig_f64(double* a, uint64_t n, double* evals) {
    return guard([&] {
        std::vector<double> m(a, a + n * n), ev;
        sym_eig(m, n, ev);
        std::memcpy(a, m.data(), n * n * sizeof(double));
        std::memcpy(evals, ev.data(), n * sizeof(double));
    });
}

int orc_quantize_method_f64(const double* core, const uint64_t* shape, int d, int method, uint64_t* mag,
                            uint8_t* neg, int* k, int* zero, double* slice_norms) {
    return guard([&] {
        const Shape sh = to_shape(shape, d);
        std::vector<double> x(core, core + numel(sh));
        const auto om = order_map(method, sh);
        auto q = quantize(x, sh, om);
        *k = q.k;
        *zero = q.zero;
        if (!q.zero) {
            std::memcpy(mag, q.mag.data(), q.mag.size() * 8);
            std::memcpy(neg, q.neg.data(), q.neg.size());
        }
        std::size_t o = 0;
        for (int a = 0; a < d; ++a)
            for (double s : q.slice_norms[a]) slice_norms[o++] = s;
    });
}

int orc_quantize_f64(const double* core, const uint64_t* shape, int d, uint64_t* mag, uint8_t* neg, int* k,
                     int* zero, double* slice_norms) {
    return orc_quantize_method_f64(core, shape, d, 0, mag, neg, k, zero, slice_norms);
}

int orc_encode(const uint64_t* m, const uint8_t* neg, uint64_t n, double target_int, int coder, uint64_t block,
               int split, int fixed_plane, uint8_t** out, uint64_t* out_len, int* last_plane, double* achieved,
               uint64_t* decoded) {
    return guard([&] {
        CodecOpts o;
        o.coder = static_cast<Coder>(coder);
        o.block = block;
        o.split = split != 0;
        if (fixed_plane >= 0) o.fixed_plane = fixed_plane;
        CoreEncoder enc({m, n}, o);
        enc.plan(target_int);
        if (decoded) std::memcpy(decoded, enc.planned().decoded.data(), n * 8);
        Stream s = enc.finalize({neg, n});
        auto b = serial(n, s);
        *out = dup(b);
        *out_len = b.size();
        *last_plane = s.last_plane;
        *achieved = s.achieved_int;
    });
}

int orc_encode_symbols(int coder, const uint64_t* s, uint64_t n, uint8_t** out, uint64_t* len) {
    return guard([&] {
        auto b = pack_symbols(static_cast<Coder>(coder), {s, n});
        *out = dup(b);
        *len = b.size();
    });
}

int orc_decode_symbols(const uint8_t* p, uint64_t len, uint64_t** out, uint64_t* n) {
    return guard([&] {
        auto v = unpack_symbols({p, len});
        *out = dup(v);
        *n = v.size();
    });
}

int orc_encode_factor_f64(const double* u, uint64_t n, uint64_t r, const uint8_t* dead, const double* sn, int coder,
                          int simple, int core_step_log2, double cap, uint8_t** stream, uint64_t* len, int* k,
                          uint64_t* count, int8_t* flips, double* term, int* plane, double* decoded) {
    return guard([&] {
        std::vector<double> uu(u, u + n * r);
        FactorOpts o;
        o.coder = static_cast<Coder>(coder);
        o.simple = simple != 0;
        o.core_step_log2 = core_step_log2;
        o.term_cap = cap;
        auto f = encode_factor(uu, n, r, {dead, r}, {sn, r}, o);
        auto b = serial(f.count, f.stream);
        *stream = dup(b);
        *len = b.size();
        *k = f.k;
        *count = f.count;
        for (uint64_t j = 0; j < r; ++j) flips[j] = f.flips[j];
        *term = f.term;
        *plane = f.plane;
        std::memcpy(decoded, f.decoded.data(), n * r * sizeof(double));
    });
}

double orc_sum_sq_f64(const double* x, uint64_t n) { return sum_sq(x, n); }
double orc_sum_sq_f32(const float* x, uint64_t n) { return sum_sq(x, n); }
double orc_backward_sq(const uint64_t* m, uint64_t n) { return backward_sq(std::span<const u64>(m, n)); }
int orc_recal_due(uint64_t terms, double ref, double running) { return recal_due(terms, ref, running); }
int orc_pick_rank(const double* s2, uint64_t n, double budget, uint64_t* r, double* discarded) {
    return guard([&] {
        auto c = pick_rank({s2, n}, budget);
        *r = c.r;
        *discarded = c.discarded;
    });
}
int orc_alpha_weights(const double* sn, uint64_t r, uint64_t n, double* out) {
    return guard([&] {
        auto a = alpha_weights({sn, r}, n);
        std::memcpy(out, a.data(), r * sizeof(double));
    });
}
int orc_transpose_f64(const double* x, const uint64_t* shape, int d, const uint64_t* perm, double* out) {
    return guard([&] {
        const Shape sh = to_shape(shape, d);
        std::vector<double> v(x, x + numel(sh));
        auto t = permute_axes(v, sh, Perm(perm, perm + d));
        std::memcpy(out, t.data(), t.size() * sizeof(double));
    });
}
}
