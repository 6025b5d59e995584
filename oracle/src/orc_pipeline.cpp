// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp).
// Restates sthosvd.cpp:13-218 (rank rule, mode order, left_svd switch, sign
// fix, circular-shift projection, reconstruction), factor_codec.cpp:19-264
// (Householder reflectors, alpha weights, plane-deepening loop),
// container.cpp:51-420 (ingest, TKC1 writer/reader) and pipeline.cpp:24-236
// (compress_impl / decompress_impl orchestration).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <type_traits>

#include "orc.hpp"

namespace orc {

namespace {
using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}
}  // namespace

// ---------------------------------------------------------------- sthosvd
RankChoice pick_rank(std::span<const double> s2, double budget) {
    if (s2.empty()) throw Error("rank choice: empty singular values");
    if (budget < 0) throw Error("rank choice: negative budget");
    std::size_t r = s2.size();
    double gone = 0.0;
    while (r > 0) {
        const double next = gone + s2[r - 1];
        if (next > budget) break;
        gone = next;
        --r;
    }
    return {r, gone};
}

namespace {

// lower triangle of B B^T (B row-major rows x cols) into column-major g
template <class T>
void gram_lower(const T* b, std::size_t rows, std::size_t cols, std::vector<T>& g) {
    g.assign(rows * rows, T(0));
    // one output per (i, j), each summed in the same order whatever the thread count
#pragma omp parallel for schedule(dynamic, 1)
    for (std::size_t j = 0; j < rows; ++j)
        for (std::size_t i = j; i < rows; ++i) {
            const T* x = b + i * cols;
            const T* y = b + j * cols;
            T s0 = 0, s1 = 0, s2 = 0, s3 = 0;
            std::size_t c = 0;
            for (; c + 4 <= cols; c += 4) {
                s0 += x[c] * y[c];
                s1 += x[c + 1] * y[c + 1];
                s2 += x[c + 2] * y[c + 2];
                s3 += x[c + 3] * y[c + 3];
            }
            for (; c < cols; ++c) s0 += x[c] * y[c];
            g[i + j * rows] = (s0 + s1) + (s2 + s3);
        }
}

}  // namespace

template <class T>
Tucker<T> sthosvd(const std::vector<T>& a, const Shape& shape, double target,
                  const std::optional<Perm>& order, SvdBackend be) {
    if (target < 0) throw Error("sthosvd: negative SSE target");
    if (!finite_all(a.data(), a.size())) throw Error("sthosvd: input contains non-finite values");
    const std::size_t d = shape.size();
    Perm p = order ? *order : stable_ascending(shape);
    if (p.size() != d || !valid_perm(p)) throw Error("sthosvd: invalid processing order");
    Tucker<T> f;
    f.order = p;
    f.factors.resize(d);
    f.trunc.assign(d, 0.0);
    f.n = shape;
    f.r.assign(d, 0);
    std::vector<T> x = permute_axes(a, shape, p);
    std::vector<std::size_t> cur(d);
    for (std::size_t i = 0; i < d; ++i) cur[i] = shape[p[i]];
    double remaining = target;
    for (std::size_t step = 0; step < d; ++step) {
        const std::size_t rows = cur[0], cols = x.size() / rows;
        std::vector<T> u;  // column-major rows x k
        std::vector<double> s2;
        const bool via_gram = be == SvdBackend::gram || (be == SvdBackend::automatic && rows <= cols);
        std::size_t ucols;
        if (via_gram) {
            std::vector<T> g, ev;
            gram_lower(x.data(), rows, cols, g);
            sym_eig(g, rows, ev);
            u.resize(rows * rows);
            s2.resize(rows);
            for (std::size_t j = 0; j < rows; ++j) {
                const std::size_t src = rows - 1 - j;
                std::copy(g.begin() + src * rows, g.begin() + (src + 1) * rows, u.begin() + j * rows);
                s2[j] = std::max(0.0, static_cast<double>(ev[src]));
            }
            ucols = rows;
        } else {
            std::vector<T> sv;
            thin_svd(x.data(), rows, cols, u, sv);
            ucols = cols;
            s2.resize(cols);
            for (std::size_t j = 0; j < cols; ++j) {
                const double s = static_cast<double>(sv[j]);
                s2[j] = s * s;
            }
        }
        f.sigma2.push_back(s2);
        const double budget = remaining / static_cast<double>(d - step);
        RankChoice ch = pick_rank(s2, budget);
        if (ch.r == 0) {  // keep one basis vector even when the budget covers everything
            ch.r = 1;
            ch.discarded -= s2[0];
        }
        (void)ucols;
        remaining = std::max(0.0, remaining - ch.discarded);
        f.trunc[p[step]] = ch.discarded;
        const std::size_t r = ch.r;
        // sign convention: each column's largest-magnitude entry (first on ties) >= 0
        for (std::size_t j = 0; j < r; ++j) {
            T* c = u.data() + j * rows;
            std::size_t im = 0;
            for (std::size_t i = 1; i < rows; ++i)
                if (std::fabs(c[i]) > std::fabs(c[im])) im = i;
            if (c[im] < T(0))
                for (std::size_t i = 0; i < rows; ++i) c[i] = -c[i];
        }
        std::vector<T> fac(rows * r);
        for (std::size_t i = 0; i < rows; ++i)
            for (std::size_t j = 0; j < r; ++j) fac[i * r + j] = u[i + j * rows];
        f.factors[p[step]] = fac;
        f.r[p[step]] = r;
        // projection fused with the circular shift: next (cols x r) = B^T U_r
        std::vector<T> nx(cols * r, T(0));
        // column ranges in parallel; every output still accumulates i = 0, 1, ... in order
        const std::size_t cb = 4096;
#pragma omp parallel for schedule(static)
        for (std::size_t c0 = 0; c0 < cols; c0 += cb) {
            const std::size_t c1 = std::min(cols, c0 + cb);
            for (std::size_t i = 0; i < rows; ++i) {
                const T* brow = x.data() + i * cols;
                const T* urow = fac.data() + i * r;
                for (std::size_t c = c0; c < c1; ++c) {
                    const T bv = brow[c];
                    T* o = nx.data() + c * r;
                    for (std::size_t j = 0; j < r; ++j) o[j] += bv * urow[j];
                }
            }
        }
        x = std::move(nx);
        cur.erase(cur.begin());
        cur.push_back(r);
    }
    f.core = std::move(x);
    f.core_shape = Shape(cur.begin(), cur.end());
    return f;
}
template Tucker<float> sthosvd(const std::vector<float>&, const Shape&, double, const std::optional<Perm>&, SvdBackend);
template Tucker<double> sthosvd(const std::vector<double>&, const Shape&, double, const std::optional<Perm>&, SvdBackend);

namespace {
Perm decompression_order(const Shape& n, const std::vector<std::size_t>& r) {
    const std::size_t d = n.size();
    if (d > 8) throw Error("mode order: exhaustive search limited to order 8");
    Perm perm(d);
    for (std::size_t i = 0; i < d; ++i) perm[i] = i;
    auto cost = [&](const Perm& q) {
        unsigned __int128 tot = 0;
        for (std::size_t i = 0; i < d; ++i) {
            unsigned __int128 t = 1;
            for (std::size_t j = 0; j <= i; ++j) t *= n[q[j]];
            for (std::size_t j = i; j < d; ++j) t *= r[q[j]];
            tot += t;
        }
        return tot;
    };
    Perm best = perm;
    auto bc = cost(perm);
    while (std::next_permutation(perm.begin(), perm.end())) {
        const auto c = cost(perm);
        if (c < bc) {
            bc = c;
            best = perm;
        }
    }
    return best;
}
}  // namespace

template <class T>
std::vector<T> tucker_expand(const Tucker<T>& f) {
    const std::size_t d = f.order.size();
    const Perm q = decompression_order(f.n, f.r);
    const Perm ip = inverse_perm(f.order);
    Perm ax(d);
    for (std::size_t j = 0; j < d; ++j) ax[j] = ip[q[j]];
    std::vector<T> x = permute_axes(f.core, f.core_shape, ax);
    std::vector<std::size_t> cur(d);
    for (std::size_t j = 0; j < d; ++j) cur[j] = f.r[q[j]];
    for (std::size_t step = 0; step < d; ++step) {
        const std::size_t mode = q[step];
        const std::size_t rows = cur[0], cols = x.size() / rows, nn = f.n[mode];
        const std::vector<T>& u = f.factors[mode];  // nn x rows, row-major
        std::vector<T> nx(cols * nn, T(0));
        for (std::size_t i = 0; i < rows; ++i)
            for (std::size_t c = 0; c < cols; ++c) {
                const T bv = x[i * cols + c];
                T* o = nx.data() + c * nn;
                for (std::size_t k = 0; k < nn; ++k) o[k] += bv * u[k * rows + i];
            }
        x = std::move(nx);
        cur.erase(cur.begin());
        cur.push_back(nn);
    }
    Shape sq(cur.begin(), cur.end());
    return permute_axes(x, sq, inverse_perm(q));
}
template std::vector<float> tucker_expand(const Tucker<float>&);
template std::vector<double> tucker_expand(const Tucker<double>&);

// ---------------------------------------------------------------- factor codec
namespace {

template <class T>
struct Householder {
    std::vector<T> refl;  // column-major n x r
    std::vector<signed char> flips;
    std::vector<T> adjusted;  // column-major n x r
};

template <class T>
Householder<T> factorize(const std::vector<T>& ucm, std::size_t n, std::size_t r) {
    if (r > n) throw Error("factorize: more columns than rows");
    if (r > 0) {
        T dev = 0;
        for (std::size_t a = 0; a < r; ++a)
            for (std::size_t b = 0; b < r; ++b) {
                T s = 0;
                for (std::size_t i = 0; i < n; ++i) s += ucm[i + a * n] * ucm[i + b * n];
                dev = std::max(dev, static_cast<T>(std::fabs(s - (a == b ? T(1) : T(0)))));
            }
        if (static_cast<double>(dev) > 1e-8) throw Error("factorize: input columns are not orthonormal");
    }
    Householder<T> h;
    h.refl.assign(n * r, T(0));
    h.flips.assign(r, 1);
    h.adjusted = ucm;
    std::vector<T> R = ucm, v(n), t(r);
    for (std::size_t i = 0; i < r; ++i) {
        const std::size_t m = n - i;
        T nrm = 0;
        for (std::size_t k = 0; k < m; ++k) v[k] = R[i + k + i * n];
        for (std::size_t k = 0; k < m; ++k) nrm += v[k] * v[k];
        nrm = std::sqrt(nrm);
        v[0] += (v[0] < T(0) ? T(-1) : T(1)) * nrm;
        T vn = 0;
        for (std::size_t k = 0; k < m; ++k) vn += v[k] * v[k];
        vn = std::sqrt(vn);
        if (vn == T(0)) throw Error("factorize: degenerate reflector");
        for (std::size_t k = 0; k < m; ++k) v[k] /= vn;
        for (std::size_t c = i; c < r; ++c) {
            T s = 0;
            for (std::size_t k = 0; k < m; ++k) s += v[k] * R[i + k + c * n];
            t[c] = s;
        }
        for (std::size_t c = i; c < r; ++c)
            for (std::size_t k = 0; k < m; ++k) R[i + k + c * n] -= T(2) * v[k] * t[c];
        if (v[0] < T(0))
            for (std::size_t k = 0; k < m; ++k) v[k] = -v[k];
        for (std::size_t k = 0; k < m; ++k) h.refl[i + k + i * n] = v[k];
        if (R[i + i * n] < T(0)) {
            h.flips[i] = -1;
            for (std::size_t k = 0; k < n; ++k) h.adjusted[k + i * n] = -h.adjusted[k + i * n];
        }
    }
    return h;
}

// product of the reflections applied to the first r identity columns
template <class T>
std::vector<T> householder_expand(std::vector<T> v, std::size_t n, std::size_t r) {
    for (std::size_t j = 0; j < r; ++j) {
        T below = 0;
        for (std::size_t i = j + 1; i < n; ++i) below += v[i + j * n] * v[i + j * n];
        if (static_cast<double>(below) >= 1.0) throw Error("reconstruct: reflector sub-diagonal norm reaches 1");
        v[j + j * n] = std::sqrt(T(1) - below);
    }
    std::vector<T> x(n * r, T(0));
    for (std::size_t j = 0; j < r; ++j) x[j + j * n] = T(1);
    std::vector<T> t(r);
    for (std::size_t j = r; j-- > 0;) {
        const T* vj = v.data() + j * n;
        for (std::size_t c = 0; c < r; ++c) {
            T s = 0;
            for (std::size_t i = j; i < n; ++i) s += vj[i] * x[i + c * n];
            t[c] = s;
        }
        for (std::size_t c = 0; c < r; ++c)
            for (std::size_t i = j; i < n; ++i) x[i + c * n] -= T(2) * vj[i] * t[c];
    }
    return x;
}

std::vector<double> column_scales(std::span<const double> sn, std::size_t n, bool simple) {
    std::vector<double> w(sn.size());
    if (simple) {
        for (std::size_t j = 0; j < sn.size(); ++j) w[j] = sn[j];
    } else {
        const auto al = alpha_weights(sn, n);
        for (std::size_t j = 0; j < sn.size(); ++j) w[j] = std::sqrt(2.0 * al[j]);
    }
    return w;
}

// decoded stream -> live factor (Householder expansion) -> full n x r, column-major
template <class T>
std::vector<T> assemble(std::size_t n, std::size_t r, std::span<const u8> dead, std::span<const double> sc,
                        std::span<const u64> mag, std::span<const u8> neg, int k) {
    std::vector<std::size_t> live;
    for (std::size_t j = 0; j < r; ++j)
        if (!dead[j]) live.push_back(j);
    const std::size_t rl = live.size();
    std::vector<T> refl(n * rl, T(0));
    std::size_t s = 0;
    for (std::size_t j = 0; j < rl; ++j)
        for (std::size_t i = j + 1; i < n; ++i, ++s) {
            double val = std::ldexp(static_cast<double>(mag[s]), -k);
            if (neg[s]) val = -val;
            refl[i + j * n] = static_cast<T>(val / sc[j]);
        }
    if (s != mag.size()) throw Error("factor decode: stream length mismatch");
    std::vector<T> full(n * r, T(0));
    if (rl > 0) {
        const auto lf = householder_expand(refl, n, rl);
        for (std::size_t j = 0; j < rl; ++j)
            std::copy(lf.begin() + j * n, lf.begin() + (j + 1) * n, full.begin() + live[j] * n);
    }
    return full;
}

template <class T>
std::vector<T> to_row_major(const std::vector<T>& cm, std::size_t n, std::size_t r) {
    std::vector<T> o(n * r);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < r; ++j) o[i * r + j] = cm[i + j * n];
    return o;
}

}  // namespace

std::vector<double> alpha_weights(std::span<const double> sn, std::size_t n) {
    const std::size_t r = sn.size();
    if (n < r) throw Error("weights: factor has more columns than rows");
    std::vector<double> al(r);
    double tail = 0.0;
    for (std::size_t k = 0; k < r; ++k) tail += sn[k] * sn[k];
    for (std::size_t j = 0; j < r; ++j) {
        const double sj = sn[j];
        tail -= sj * sj;
        const double nj = static_cast<double>(n - j);
        const double q = std::sqrt(nj);
        al[j] = (1.0 + (nj + 5.0 * q + 2.0) / ((q + 1.0) * (q + 1.0) * q)) * sj * sj;
        if (tail > 0.0)
            al[j] += (2.0 / (nj - 1.0) + (nj + 2.0 * q + 2.0) / ((q + 1.0) * (q + 1.0) * (q + 1.0) * q)) * tail;
    }
    return al;
}

template <class T>
FactorOut<T> encode_factor(const std::vector<T>& u, std::size_t n, std::size_t r, std::span<const u8> dead,
                           std::span<const double> sn, const FactorOpts& o) {
    if (dead.size() != r || sn.size() != r) throw Error("factor encode: column metadata mismatch");
    FactorOut<T> out;
    out.dead.assign(dead.begin(), dead.end());
    out.flips.assign(r, 1);
    std::vector<std::size_t> live;
    std::vector<double> ln;
    for (std::size_t j = 0; j < r; ++j)
        if (!dead[j]) {
            live.push_back(j);
            ln.push_back(sn[j]);
        }
    const std::size_t rl = live.size();
    if (rl == 0) {  // stream stays default: block 0, no planes (factor_codec.cpp:174-177)
        out.decoded.assign(n * r, T(0));
        return out;
    }
    std::vector<T> ul(n * rl);  // column-major live columns
    for (std::size_t j = 0; j < rl; ++j)
        for (std::size_t i = 0; i < n; ++i) ul[i + j * n] = u[i * r + live[j]];
    const auto h = factorize(ul, n, rl);
    for (std::size_t j = 0; j < rl; ++j) out.flips[live[j]] = h.flips[j];
    const auto sc = column_scales(ln, n, o.simple);
    out.count = n * rl - rl * (rl + 1) / 2;
    std::vector<double> st;
    st.reserve(out.count);
    for (std::size_t j = 0; j < rl; ++j)
        for (std::size_t i = j + 1; i < n; ++i) st.push_back(static_cast<double>(h.refl[i + j * n]) * sc[j]);
    const double mx = st.empty() ? 0.0 : max_abs_d(st.data(), st.size());
    out.k = mx > 0.0 ? 63 - std::ilogb(mx) : 0;
    std::vector<u64> mag(st.size());
    std::vector<u8> neg(st.size());
    for (std::size_t s = 0; s < st.size(); ++s) {
        mag[s] = static_cast<u64>(std::nearbyint(std::ldexp(std::fabs(st[s]), out.k)));
        neg[s] = st[s] < 0 ? 1 : 0;
    }
    int plane = std::clamp(o.core_step_log2 + out.k, 0, 63);
    std::vector<T> adj(n * r, T(0));  // column-major
    for (std::size_t j = 0; j < rl; ++j)
        std::copy(h.adjusted.begin() + j * n, h.adjusted.begin() + (j + 1) * n, adj.begin() + live[j] * n);
    while (true) {
        CodecOpts eo;
        eo.coder = o.coder;
        eo.split = false;
        eo.fixed_plane = plane;
        CoreEncoder enc(mag, eo);
        enc.plan(0.0);
        const auto full = assemble<T>(n, r, dead, sc, enc.planned().decoded, neg, out.k);
        out.term = 0.0;
        for (std::size_t j = 0; j < rl; ++j) {
            T s = 0;
            for (std::size_t i = 0; i < n; ++i) {
                const T dlt = full[i + live[j] * n] - adj[i + live[j] * n];
                s += dlt * dlt;
            }
            out.term += ln[j] * ln[j] * static_cast<double>(s);
        }
        if (out.term <= o.term_cap || plane == 0) {
            out.stream = enc.finalize(neg);
            out.decoded = to_row_major(full, n, r);
            out.plane = plane;
            return out;
        }
        const double excess = out.term / std::max(o.term_cap, 1e-300);
        const int step = std::max(1, static_cast<int>(std::ceil(0.25 * std::log2(excess))));
        plane = std::max(0, plane - step);
    }
}
template FactorOut<float> encode_factor(const std::vector<float>&, std::size_t, std::size_t, std::span<const u8>,
                                        std::span<const double>, const FactorOpts&);
template FactorOut<double> encode_factor(const std::vector<double>&, std::size_t, std::size_t, std::span<const u8>,
                                         std::span<const double>, const FactorOpts&);

template <class T>
std::vector<T> decode_factor(std::size_t n, std::size_t r, std::span<const u8> dead, std::span<const double> sn,
                             bool simple, int k, u64 count, const StreamMeta& meta,
                             const std::vector<std::vector<std::span<const u8>>>& pl) {
    std::vector<double> ln;
    for (std::size_t j = 0; j < r; ++j)
        if (!dead[j]) ln.push_back(sn[j]);
    if (ln.empty()) return std::vector<T>(n * r, T(0));
    if (count != n * ln.size() - ln.size() * (ln.size() + 1) / 2)
        throw Error("factor decode: coefficient count mismatch");
    const auto sc = column_scales(ln, n, simple);
    const auto dec = decode_stream(meta, pl);
    return to_row_major(assemble<T>(n, r, dead, sc, dec.mag, dec.neg, k), n, r);
}
template std::vector<float> decode_factor(std::size_t, std::size_t, std::span<const u8>, std::span<const double>, bool,
                                          int, u64, const StreamMeta&,
                                          const std::vector<std::vector<std::span<const u8>>>&);
template std::vector<double> decode_factor(std::size_t, std::size_t, std::span<const u8>, std::span<const double>,
                                           bool, int, u64, const StreamMeta&,
                                           const std::vector<std::vector<std::span<const u8>>>&);

// ---------------------------------------------------------------- container
std::size_t dtype_bytes(Dtype t) {
    switch (t) {
        case Dtype::i8: case Dtype::u8_: return 1;
        case Dtype::i16: case Dtype::u16: return 2;
        case Dtype::i32: case Dtype::u32_: case Dtype::f32: return 4;
        case Dtype::i64: case Dtype::u64_: case Dtype::f64: return 8;
    }
    throw Error("container: unknown dtype");
}

namespace {

template <class N, class T>
void cast_in(std::span<const u8> raw, std::vector<T>& out, bool& loss) {
    const std::size_t n = raw.size() / sizeof(N);
    out.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
        N v;
        std::memcpy(&v, raw.data() + i * sizeof(N), sizeof(N));
        out[i] = static_cast<T>(v);
        if constexpr (std::is_integral_v<N> && sizeof(N) == 8) {
            const auto mag = static_cast<u64>(v < 0 ? -(v + 1) : v);
            if (mag > (u64{1} << 53)) loss = true;
        }
    }
}

template <class T>
std::vector<T> ingest(std::span<const u8> bytes, Dtype dt, const Shape& shape, std::size_t skip, bool& loss) {
    const u64 n = numel(shape);
    const std::size_t expect = skip + n * dtype_bytes(dt);
    if (bytes.size() != expect)
        throw Error("ingest: buffer holds " + std::to_string(bytes.size()) + " bytes, expected " +
                    std::to_string(expect));
    for (auto s : shape)
        if (s == 0) throw Error("tensor: zero-sized mode");
    std::vector<T> v;
    const auto raw = bytes.subspan(skip);
    switch (dt) {
        case Dtype::i8: cast_in<std::int8_t>(raw, v, loss); break;
        case Dtype::u8_: cast_in<std::uint8_t>(raw, v, loss); break;
        case Dtype::i16: cast_in<std::int16_t>(raw, v, loss); break;
        case Dtype::u16: cast_in<std::uint16_t>(raw, v, loss); break;
        case Dtype::i32: cast_in<std::int32_t>(raw, v, loss); break;
        case Dtype::u32_: cast_in<std::uint32_t>(raw, v, loss); break;
        case Dtype::i64: cast_in<std::int64_t>(raw, v, loss); break;
        case Dtype::u64_: cast_in<std::uint64_t>(raw, v, loss); break;
        case Dtype::f32: cast_in<float>(raw, v, loss); break;
        case Dtype::f64: cast_in<double>(raw, v, loss); break;
    }
    return v;
}

struct W {
    Bytes b;
    void u8v(u8 v) { b.push_back(v); }
    void u32v(u32 v) {
        for (int i = 0; i < 4; ++i) b.push_back(static_cast<u8>(v >> (8 * i)));
    }
    void u64v(u64 v) {
        for (int i = 0; i < 8; ++i) b.push_back(static_cast<u8>(v >> (8 * i)));
    }
    void f64v(double v) {
        u64 x;
        std::memcpy(&x, &v, 8);
        u64v(x);
    }
    void raw(const Bytes& x) { b.insert(b.end(), x.begin(), x.end()); }
};

void put_stream(W& w, u64 count, const Stream& s) {
    w.u64v(count);
    w.u64v(s.block);
    w.u8v(static_cast<u8>(s.last_plane));
    w.u32v(static_cast<u32>(s.stops.size()));
    for (const auto& st : s.stops) {
        w.u64v(st.lead);
        w.u64v(st.trail);
    }
    w.u32v(static_cast<u32>(s.payloads.size()));
    for (const auto& pl : s.payloads)
        for (const auto& blk : pl) {
            w.u32v(static_cast<u32>(blk.size()));
            w.raw(blk);
        }
}

struct R {
    std::span<const u8> b;
    std::size_t pos = 0;
    std::string sec;
    void need(std::size_t n) const {
        if (pos + n > b.size()) throw Error("container: truncated " + sec + " section");
    }
    u8 u8v() {
        need(1);
        return b[pos++];
    }
    u32 u32v() {
        need(4);
        u32 v = 0;
        for (int i = 0; i < 4; ++i) v |= static_cast<u32>(b[pos + i]) << (8 * i);
        pos += 4;
        return v;
    }
    u64 u64v() {
        need(8);
        u64 v = 0;
        for (int i = 0; i < 8; ++i) v |= static_cast<u64>(b[pos + i]) << (8 * i);
        pos += 8;
        return v;
    }
    double f64v() {
        const u64 x = u64v();
        double v;
        std::memcpy(&v, &x, 8);
        return v;
    }
    std::span<const u8> raw(std::size_t n) {
        need(n);
        auto s = b.subspan(pos, n);
        pos += n;
        return s;
    }
};

struct StreamView {
    StreamMeta meta;
    std::vector<std::vector<std::span<const u8>>> pl;
};

StreamView get_stream(R& r) {
    StreamView v;
    v.meta.count = r.u64v();
    v.meta.block = r.u64v();
    v.meta.last_plane = r.u8v();
    const u32 nb = r.u32v();
    v.meta.stops.resize(nb);
    for (auto& s : v.meta.stops) {
        s.lead = r.u64v();
        s.trail = r.u64v();
    }
    const u32 np = r.u32v();
    if (np > 64) throw Error("container: implausible plane count");
    v.pl.assign(np, {});
    for (auto& row : v.pl) {
        row.resize(nb);
        for (auto& blk : row) blk = r.raw(r.u32v());
    }
    return v;
}

struct Header {
    Dtype dt = Dtype::f64;
    bool f32 = false;
    std::vector<u64> n, r;
    Perm order, storage;
    Coder coder = Coder::ac;
    u8 method = 0;
    bool zero = false, split = true, simple = false;
    int k = 0;
    u64 block = 0;
    double rtmss = 0.5, target = 0, norm = 0, trunc = 0, cq = 0, est = 0;
};

struct FactorPayload {
    std::vector<u8> dead;
    std::vector<double> sn;
    int k = 0;
    u64 count = 0;
    Stream stream;
};

Bytes write_container(const Header& h, const std::vector<FactorPayload>& fs, const Stream& core) {
    const std::size_t d = h.n.size();
    if (!h.zero && fs.size() != d) throw Error("container: factor payload count mismatch");
    W w;
    w.raw(Bytes{'T', 'K', 'C', '1'});
    w.u8v(1);
    w.u8v(static_cast<u8>(h.dt));
    w.u8v(h.f32 ? 1 : 0);
    w.u8v(static_cast<u8>(d));
    w.u8v(static_cast<u8>(h.coder));
    w.u8v(h.method);
    w.u8v(static_cast<u8>((h.zero ? 1 : 0) | (h.split ? 2 : 0) | (h.simple ? 4 : 0)));
    w.u8v(0);
    for (auto v : h.n) w.u64v(v);
    for (auto v : h.r) w.u64v(v);
    for (auto v : h.order) w.u8v(static_cast<u8>(v));
    for (auto v : h.storage) w.u8v(static_cast<u8>(v));
    w.u32v(static_cast<u32>(h.k));
    w.u64v(h.block);
    for (double v : {h.rtmss, h.target, h.norm, h.trunc, h.cq, h.est}) w.f64v(v);
    if (!h.zero) {
        for (const auto& f : fs) {
            W fw;
            const std::size_t r = f.sn.size();
            for (std::size_t j = 0; j < r; j += 8) {
                u8 bits = 0;
                for (std::size_t q = 0; q < 8 && j + q < r; ++q)
                    if (f.dead[j + q]) bits |= static_cast<u8>(1u << q);
                fw.u8v(bits);
            }
            for (double s : f.sn) fw.f64v(s);
            fw.u32v(static_cast<u32>(f.k));
            fw.u64v(f.count);
            put_stream(fw, f.count, f.stream);
            w.u64v(fw.b.size());
            w.raw(fw.b);
        }
        u64 cnt = 1;
        for (auto v : h.r) cnt *= v;
        W cw;
        put_stream(cw, cnt, core);
        w.u64v(cw.b.size());
        w.raw(cw.b);
    }
    return std::move(w.b);
}

template <class T>
Result compress_as(std::vector<T> a, const Shape& shape, Dtype dt, const Params& prm) {
    const auto t_all = Clock::now();
    Result res;
    res.original_bytes = a.size() * dtype_bytes(dt);
    const std::size_t d = shape.size();
    if (prm.target_re && prm.target_sse)
        throw Error("compress: relative-error and SSE targets are mutually exclusive");
    if (!prm.target_re && !prm.target_sse) throw Error("compress: no error target given");
    res.norm_sq = sum_sq(a.data(), a.size());
    double target;
    if (prm.target_re) {
        if (*prm.target_re < 0) throw Error("budget: negative relative-error target");
        target = *prm.target_re * *prm.target_re * res.norm_sq;
    } else {
        target = *prm.target_sse;
    }
    if (target < 0) throw Error("budget: negative SSE target");
    if (prm.rtmss < 0 || prm.rtmss > 1) throw Error("budget: rtmss outside [0, 1]");
    res.target_sse = target;
    auto t0 = Clock::now();
    Tucker<T> f = sthosvd(a, shape, prm.rtmss * target, prm.mode_order, prm.backend);
    double trunc = 0;
    for (double v : f.trunc) trunc += v;
    double core_target = target - trunc;
    if (core_target < 0) core_target = 0;
    res.t_sthosvd = ms_since(t0);
    a.clear();
    a.shrink_to_fit();

    Header h;
    h.dt = dt;
    h.f32 = std::is_same_v<T, float>;
    h.n.assign(shape.begin(), shape.end());
    h.r.assign(f.r.begin(), f.r.end());
    h.order = f.order;
    h.coder = prm.coder;
    h.split = prm.split;
    h.simple = prm.simple;
    h.rtmss = prm.rtmss;
    h.target = target;
    h.norm = res.norm_sq;
    h.trunc = trunc;
    res.ranks = h.r;
    res.trunc = trunc;

    t0 = Clock::now();
    Perm storage = prm.storage_order ? *prm.storage_order : stable_ascending(f.core_shape);
    if (storage.size() != d || !valid_perm(storage)) throw Error("compress: invalid storage order");
    h.storage = storage;
    Shape cs(d);
    for (std::size_t i = 0; i < d; ++i) cs[i] = f.core_shape[storage[i]];
    std::vector<T> core_s = permute_axes(f.core, f.core_shape, storage);
    const std::vector<u64> vorder = order_map(prm.method, cs);  // vectorize::OrderMap::build (pipeline.cpp:87)
    h.method = static_cast<u8>(prm.method);
    Quantized q = quantize(core_s, cs, vorder);
    core_s.clear();
    res.t_quant = ms_since(t0);
    h.zero = q.zero;
    h.k = q.k;
    res.core_k = q.k;
    h.block = prm.block ? prm.block : default_block(q.mag.size());
    if (q.zero) {
        res.estimate = trunc;
        h.cq = 0;
        h.est = trunc;
        res.container = write_container(h, {}, Stream{});
        res.t_total = ms_since(t_all);
        return res;
    }
    std::vector<std::size_t> mode_of(d);
    for (std::size_t ax = 0; ax < d; ++ax) mode_of[ax] = f.order[storage[ax]];
    std::vector<std::vector<double>> sn_mode(d);
    for (std::size_t ax = 0; ax < d; ++ax) sn_mode[mode_of[ax]] = q.slice_norms[ax];

    t0 = Clock::now();
    CodecOpts co;
    co.coder = prm.coder;
    co.block = h.block;
    co.split = prm.split;
    CoreEncoder enc(q.mag, co);
    enc.plan(std::ldexp(core_target, 2 * q.k));
    res.t_core = ms_since(t0);
    res.core_last_plane = enc.planned().last_plane;
    const auto dead_ax = dead_slices(cs, enc.planned().decoded, vorder);
    std::vector<std::vector<u8>> dead_mode(d);
    for (std::size_t ax = 0; ax < d; ++ax) dead_mode[mode_of[ax]] = dead_ax[ax];

    t0 = Clock::now();
    FactorOpts fo;
    fo.coder = prm.coder;
    fo.simple = prm.simple;
    fo.core_step_log2 = enc.planned().last_plane - q.k;
    fo.term_cap = 0.02 * target / static_cast<double>(d);
    std::vector<FactorPayload> fp(d);
    std::vector<std::vector<signed char>> flips(d);
    res.factor_terms.assign(d, 0.0);
    for (std::size_t i = 0; i < d; ++i) {
        auto ef = encode_factor(f.factors[i], f.n[i], f.r[i], dead_mode[i], sn_mode[i], fo);
        flips[i] = ef.flips;
        res.factor_terms[i] = ef.term;
        fp[i].dead = ef.dead;
        fp[i].sn = sn_mode[i];
        fp[i].k = ef.k;
        fp[i].count = ef.count;
        fp[i].stream = std::move(ef.stream);
    }
    res.t_factor = ms_since(t0);

    t0 = Clock::now();
    const auto st = strides_of(cs);
    std::vector<u8> neg = q.neg;
    for (std::size_t v = 0; v < neg.size(); ++v) {
        const u64 pos = vorder.empty() ? v : vorder[v];
        u8 par = 0;
        for (std::size_t ax = 0; ax < d; ++ax)
            if (flips[mode_of[ax]][(pos / st[ax]) % cs[ax]] < 0) par ^= 1;
        neg[v] ^= par;
    }
    Stream cst = enc.finalize(neg);
    res.t_core += ms_since(t0);
    res.core_quant = std::ldexp(cst.achieved_int, -2 * q.k);
    h.cq = res.core_quant;
    double est = trunc + res.core_quant;
    for (double v : res.factor_terms) est += v;
    h.est = est;
    res.estimate = est;
    t0 = Clock::now();
    res.container = write_container(h, fp, cst);
    res.t_ser = ms_since(t0);
    res.t_total = ms_since(t_all);
    return res;
}

}  // namespace

Result compress(std::span<const u8> bytes, Dtype dt, const Shape& shape, std::size_t skip, const Params& p) {
    bool loss = false;
    Result r;
    if (p.f32) {
        auto a = ingest<float>(bytes, dt, shape, skip, loss);
        r = compress_as<float>(std::move(a), shape, dt, p);
    } else {
        auto a = ingest<double>(bytes, dt, shape, skip, loss);
        r = compress_as<double>(std::move(a), shape, dt, p);
    }
    r.precision_loss = loss;
    return r;
}

template <class T>
std::vector<T> decompress_tensor(std::span<const u8> cont, Shape& shape_out) {
    R r{cont, 0, "header"};
    const auto mg = r.raw(4);
    if (std::memcmp(mg.data(), "TKC1", 4) != 0) throw Error("container: bad magic");
    const int version = r.u8v();
    if (version != 1) throw Error("container: unsupported format version " + std::to_string(version));
    Header h;
    h.dt = static_cast<Dtype>(r.u8v());
    if (static_cast<int>(h.dt) > 9) throw Error("container: unknown source dtype");
    h.f32 = r.u8v() != 0;
    const std::size_t d = r.u8v();
    if (d == 0) throw Error("container: zero tensor order");
    const int coder = r.u8v();
    if (coder > 1) throw Error("container: unknown entropy coder id");
    h.coder = static_cast<Coder>(coder);
    h.method = r.u8v();
    if (h.method > 2) throw Error("container: unknown vectorization method id");
    const u8 fl = r.u8v();
    h.zero = fl & 1;
    h.simple = fl & 4;
    r.u8v();
    h.n.resize(d);
    h.r.resize(d);
    for (auto& v : h.n) v = r.u64v();
    for (auto& v : h.r) v = r.u64v();
    h.order.resize(d);
    h.storage.resize(d);
    for (auto& v : h.order) v = r.u8v();
    for (auto& v : h.storage) v = r.u8v();
    // read_container's checks (container.cpp:338-420)
    auto is_perm = [d](const Perm& p) {
        std::vector<char> seen(d, 0);
        for (auto v : p) {
            if (v >= d || seen[v]) return false;
            seen[v] = 1;
        }
        return true;
    };
    if (!is_perm(h.order) || !is_perm(h.storage)) throw Error("container: corrupt mode permutations");
    for (std::size_t i = 0; i < d; ++i)
        if (h.n[i] == 0 || h.r[i] == 0 || h.r[i] > h.n[i]) throw Error("container: corrupt mode sizes or ranks");
    h.k = static_cast<std::int32_t>(r.u32v());
    h.block = r.u64v();
    for (int i = 0; i < 6; ++i) r.f64v();
    if (h.f32 != std::is_same_v<T, float>)
        throw Error("decompress: container precision does not match the requested type");
    shape_out.assign(h.n.begin(), h.n.end());
    if (h.zero) return std::vector<T>(numel(shape_out), T(0));
    Tucker<T> f;
    f.order = h.order;
    f.n.assign(h.n.begin(), h.n.end());
    f.r.assign(h.r.begin(), h.r.end());
    f.factors.resize(d);
    for (std::size_t i = 0; i < d; ++i) {
        const u64 len = r.u64v();
        R fr{r.raw(len), 0, "factor " + std::to_string(i + 1)};
        const std::size_t rk = h.r[i];
        std::vector<u8> dead(rk, 0);
        for (std::size_t j = 0; j < rk; j += 8) {
            const u8 b = fr.u8v();
            for (std::size_t q = 0; q < 8 && j + q < rk; ++q) dead[j + q] = (b >> q) & 1;
        }
        std::vector<double> sn(rk);
        for (auto& s : sn) s = fr.f64v();
        const int k = static_cast<std::int32_t>(fr.u32v());
        const u64 cnt = fr.u64v();
        auto sv = get_stream(fr);
        if (sv.meta.count != cnt) throw Error("container: factor stream length mismatch");
        f.factors[i] = decode_factor<T>(h.n[i], rk, dead, sn, h.simple, k, cnt, sv.meta, sv.pl);
    }
    const u64 len = r.u64v();
    R cr{r.raw(len), 0, "core"};
    auto cv = get_stream(cr);
    Shape cp(d), cs(d);
    for (std::size_t j = 0; j < d; ++j) cp[j] = h.r[h.order[j]];
    for (std::size_t a = 0; a < d; ++a) cs[a] = cp[h.storage[a]];
    if (cv.meta.count != numel(cs)) throw Error("container: core length does not match ranks");
    const auto dec = decode_stream(cv.meta, cv.pl);
    const std::vector<u64> vorder = order_map(h.method, cs);
    std::vector<T> core_s(numel(cs));
    for (std::size_t v = 0; v < core_s.size(); ++v) {
        double val = std::ldexp(static_cast<double>(dec.mag[v]), -h.k);
        if (dec.neg[v]) val = -val;
        core_s[vorder.empty() ? v : vorder[v]] = static_cast<T>(val);
    }
    f.core = permute_axes(core_s, cs, inverse_perm(h.storage));
    f.core_shape = cp;
    return tucker_expand(f);
}
template std::vector<float> decompress_tensor(std::span<const u8>, Shape&);
template std::vector<double> decompress_tensor(std::span<const u8>, Shape&);

}  // namespace orc
