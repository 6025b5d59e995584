// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp).
// Restates /root/reference/proj/src/core_codec.cpp (quantize :55-93, Encoder
// :105-413, decode :421-508, dead_slices :510-523) and error_model.cpp
// (:34-72).  All statistics use separate multiply/subtract/add in double with
// no contraction (this TU is built with -ffp-contract=off), exactly like the
// reference's x86-64 build without -march.
#include <algorithm>
#include <bit>
#include <cmath>

#include "orc.hpp"

namespace orc {

namespace {

inline double dbl(u64 v) { return static_cast<double>(v); }

// residual of a significant coefficient once planes >= p are known and the
// midpoint correction applies (core_codec.cpp:20-30)
inline double resid(u64 m, int p) {
    if (p == 0) return 0.0;
    const u64 below = m & ((u64{1} << p) - 1);
    return dbl(below) - dbl(u64{1} << (p - 1));
}
inline double sig2(u64 m, int p) {
    const double r = resid(m, p);
    return r * r;
}
inline double insig2(u64 m) {
    const double v = dbl(m);
    return v * v;
}
inline double trail_gain(u64 m, int p) { return sig2(m, p + 1) - sig2(m, p); }
inline double lead_gain(u64 m, int p) { return insig2(m) - sig2(m, p); }

void put_le32(Bytes& o, u32 v) {
    for (int i = 0; i < 4; ++i) o.push_back(static_cast<u8>(v >> (8 * i)));
}

}  // namespace

// ---------------------------------------------------------------- error model
double backward_sq(std::span<const u64> v) {
    double s = 0.0;
    for (std::size_t i = v.size(); i-- > 0;) {
        const double x = dbl(v[i]);
        s += x * x;
    }
    return s;
}
double backward_sq(std::span<const double> v) {
    double s = 0.0;
    for (std::size_t i = v.size(); i-- > 0;) s += v[i] * v[i];
    return s;
}
bool recal_due(u64 terms, double ref, double running) {
    const double margin = 4.0 * 2.220446049250313e-16 * static_cast<double>(terms) * ref;
    return margin > 0.1 * running;
}
double recal_sse(std::span<const u64> m, int plane) {
    if (plane < 0 || plane > 64) throw Error("recalibrate: plane out of range");
    double s = 0.0;
    for (std::size_t i = m.size(); i-- > 0;) {
        double r;
        if (plane >= 64 || (m[i] >> plane) == 0) r = dbl(m[i]);
        else if (plane == 0) r = 0.0;
        else r = dbl(m[i] & ((u64{1} << plane) - 1)) - dbl(u64{1} << (plane - 1));
        s += r * r;
    }
    return s;
}

// ---------------------------------------------------------------- quantize
template <class T>
Quantized quantize(const std::vector<T>& core, const Shape& shape, std::span<const u64> order) {
    const std::size_t n = core.size();
    if (!order.empty() && order.size() != n) throw Error("quantize: order map does not match core");
    if (numel(shape) != n) throw Error("quantize: order map does not match core");
    if (!finite_all(core.data(), n)) throw Error("quantize: non-finite core values");
    Quantized q;
    q.shape = shape;
    q.slice_norms.resize(shape.size());
    for (std::size_t a = 0; a < shape.size(); ++a) q.slice_norms[a].assign(shape[a], 0.0);
    double mx;
    if constexpr (std::is_same_v<T, float>) mx = static_cast<double>(max_abs_f(core.data(), n));
    else mx = max_abs_d(core.data(), n);
    if (mx == 0.0) {
        q.zero = true;
        return q;
    }
    q.k = 63 - std::ilogb(mx);
    const auto st = strides_of(shape);
    q.mag.resize(n);
    q.neg.resize(n);
    for (std::size_t v = 0; v < n; ++v) {
        const u64 pos = order.empty() ? v : order[v];
        const double x = static_cast<double>(core[pos]);
        const u64 m = static_cast<u64>(std::nearbyint(std::ldexp(std::fabs(x), q.k)));
        q.mag[v] = m;
        q.neg[v] = x < 0 ? 1 : 0;
        const double sq = dbl(m) * dbl(m);
        for (std::size_t a = 0; a < shape.size(); ++a) q.slice_norms[a][(pos / st[a]) % shape[a]] += sq;
    }
    const double down = std::ldexp(1.0, -2 * q.k);
    for (auto& ax : q.slice_norms)
        for (double& s : ax) s = std::sqrt(s * down);
    return q;
}
template Quantized quantize(const std::vector<float>&, const Shape&, std::span<const u64>);
template Quantized quantize(const std::vector<double>&, const Shape&, std::span<const u64>);

// ---------------------------------------------------------------- vectorization order
// Restates vectorize::PositionIterator (vectorize.cpp:40-135): zigzag walks the
// anti-diagonal layers (coordinate sum 0, 1, ...) and inside a layer moves to the
// next composition in lexicographic order; zorder visits Morton keys (axis 0
// most significant inside each bit level) in increasing order, skipping the
// subcubes that leave the shape.
std::vector<u64> order_map(int method, const Shape& shape) {
    if (method == 0) return {};
    if (method != 1 && method != 2) throw Error("vectorize: unknown method");
    const std::size_t d = shape.size();
    if (d == 0) throw Error("vectorize: empty shape");
    const auto st = strides_of(shape);
    const u64 n = numel(shape);
    std::vector<u64> out;
    out.reserve(n);
    std::vector<std::size_t> pos(d, 0);
    auto flat = [&] {
        u64 f = 0;
        for (std::size_t i = 0; i < d; ++i) f += pos[i] * st[i];
        return f;
    };
    if (method == 1) {
        std::size_t layer_max = 0, layer = 0;
        for (auto v : shape) layer_max += v - 1;
        while (true) {
            out.push_back(flat());
            bool moved = false;
            std::size_t tail = 0;
            for (std::size_t i = d - 1; i-- > 0;) {
                tail += pos[i + 1];
                if (tail >= 1 && pos[i] + 1 <= shape[i] - 1) {
                    ++pos[i];
                    std::size_t rem = tail - 1;
                    for (std::size_t j = d; j-- > i + 1;) {
                        pos[j] = std::min(rem, shape[j] - 1);
                        rem -= pos[j];
                    }
                    moved = true;
                    break;
                }
            }
            if (moved) continue;
            if (++layer > layer_max) break;
            std::size_t rem = layer;
            for (std::size_t j = d; j-- > 0;) {
                pos[j] = std::min(rem, shape[j] - 1);
                rem -= pos[j];
            }
        }
        return out;
    }
    unsigned levels = 0;
    for (auto v : shape) {
        unsigned b = 0;
        while ((u64{1} << b) < v) ++b;
        levels = std::max(levels, b);
    }
    if (static_cast<u64>(levels) * d > 63) throw Error("vectorize: shape too large for 64-bit Morton keys");
    const u64 key_end = u64{1} << (levels * d);
    for (u64 key = 0; key < key_end;) {
        bool ok = true;
        for (std::size_t a = 0; a < d && ok; ++a) {
            u64 c = 0;
            for (unsigned t = levels; t-- > 0;) c = (c << 1) | ((key >> (t * d + (d - 1 - a))) & 1u);
            if (c >= shape[a]) {
                const u64 bad = c ^ (shape[a] - 1);
                const unsigned t = 63u - static_cast<unsigned>(__builtin_clzll(bad));
                const unsigned g = t * static_cast<unsigned>(d) + static_cast<unsigned>(d - 1 - a);
                key = (key | ((u64{1} << g) - 1)) + 1;
                ok = false;
            } else {
                pos[a] = static_cast<std::size_t>(c);
            }
        }
        if (!ok) continue;
        out.push_back(flat());
        ++key;
    }
    return out;
}

// ---------------------------------------------------------------- encoder
u64 default_block(u64 n) { return std::max<u64>(4096, (n + 63) / 64); }

u64 Stream::payload_bytes() const {
    u64 t = 0;
    for (const auto& pl : payloads)
        for (const auto& b : pl) t += b.size();
    return t;
}

CoreEncoder::CoreEncoder(std::span<const u64> m, const CodecOpts& o) : m_(m), o_(o) {
    bs_ = o_.block ? o_.block : default_block(m_.size());
    nb_ = m_.empty() ? 0 : (m_.size() + bs_ - 1) / bs_;
    top_.resize(m_.size());
    for (std::size_t i = 0; i < m_.size(); ++i)
        top_[i] = m_[i] ? static_cast<signed char>(63 - std::countl_zero(m_[i])) : -1;
}

std::size_t CoreEncoder::hi_of(std::size_t b) const {
    return std::min<std::size_t>(lo_of(b) + bs_, m_.size());
}

// One (plane, block) payload: u32 entropy length, the entropy-coded zero runs
// of the leading-bit column, then the raw refinement/sign bits
// (core_codec.cpp:120-171).
Bytes CoreEncoder::emit(int p, std::size_t b, u64 lead_stop, u64 trail_stop, const u8* neg,
                        Tally* t) const {
    std::vector<u8> col;
    BitSink raw;
    u64 nl = 0, nt = 0;
    for (std::size_t i = lo_of(b), e = hi_of(b); i < e; ++i) {
        const int top = top_[i];
        if (top > p) {
            if (nt >= trail_stop) continue;
            raw.put((m_[i] >> p) & 1u);
            ++nt;
            if (t) {
                t->red_trail += trail_gain(m_[i], p);
                ++t->trail;
            }
        } else if (nl < lead_stop) {
            const bool one = top == p;
            col.push_back(one ? 1 : 0);
            ++nl;
            if (t) ++t->lead;
            if (one) {
                raw.put(neg ? neg[i] != 0 : false);
                if (t) {
                    t->red_lead += lead_gain(m_[i], p);
                    ++t->ones;
                }
            }
        }
    }
    Bytes ent;
    if (!col.empty()) ent = pack_symbols(o_.coder, zero_runs(col));
    if (t) t->ebits = ent.size() * 8;
    Bytes out;
    put_le32(out, static_cast<u32>(ent.size()));
    out.insert(out.end(), ent.begin(), ent.end());
    out.insert(out.end(), raw.bytes().begin(), raw.bytes().end());
    return out;
}

void CoreEncoder::plan(double target) {
    if (done_) throw Error("core codec: plan called twice");
    done_ = true;
    plan_.stops.assign(nb_, Stops{});
    if (m_.empty()) {
        plan_.last_plane = 63;
        decode_model();
        return;
    }
    double tracked = backward_sq(m_);
    double ref = tracked;
    u64 terms = 0;
    const int floor_p = o_.fixed_plane ? *o_.fixed_plane : 0;
    const bool budgeted = !o_.fixed_plane;
    if (budgeted && tracked <= target) {
        plan_.last_plane = 63;
        decode_model();
        return;
    }
    std::vector<Tally> per(nb_);
    Tally prev;
    bool have_prev = false;
    for (int p = 63; p >= floor_p; --p) {
        for (std::size_t b = 0; b < nb_; ++b) {
            per[b] = Tally{};
            emit(p, b, kFull, kFull, nullptr, &per[b]);
        }
        Tally tot;
        for (const auto& s : per) {
            tot.red_lead += s.red_lead;
            tot.red_trail += s.red_trail;
            tot.lead += s.lead;
            tot.ones += s.ones;
            tot.trail += s.trail;
            tot.ebits += s.ebits;
        }
        const double red = tot.red_lead + tot.red_trail;
        ++plan_.n_planes;
        if (budgeted && tracked - red <= target) {
            plan_.last_plane = p;
            stops_at(p, tracked - target, tot, per, have_prev ? &prev : nullptr);
            decode_model();
            return;
        }
        tracked -= red;
        plan_.trace.emplace_back(p, tracked);
        terms += tot.ones + tot.trail;
        if (recal_due(terms, ref, tracked)) {
            tracked = recal_sse(m_, p);
            ref = tracked;
            terms = 0;
            plan_.trace.back().second = tracked;
        }
        prev = tot;
        have_prev = true;
    }
    plan_.last_plane = floor_p;
    for (auto& s : plan_.stops) s = Stops{kFull, kFull};
    decode_model();
}

// Breakpoint plane bit placement (core_codec.cpp:252-342).
void CoreEncoder::stops_at(int p, double need, const Tally& tot, const std::vector<Tally>& per,
                           const Tally* prev) {
    auto& st = plan_.stops;
    bool lead_first = true;
    if (o_.split && prev) {
        const double lc = static_cast<double>(prev->ebits + prev->ones);
        const double tc = static_cast<double>(prev->trail);
        const double el = lc > 0 ? prev->red_lead / lc : (prev->red_lead > 0 ? HUGE_VAL : 0.0);
        const double et = tc > 0 ? prev->red_trail / tc : (prev->red_trail > 0 ? HUGE_VAL : 0.0);
        lead_first = el >= et;
    }
    if (!o_.split) {
        double cum = 0;
        std::size_t b = 0;
        for (; b < nb_; ++b) {
            const double br = per[b].red_lead + per[b].red_trail;
            if (cum + br >= need) break;
            cum += br;
            st[b] = {kFull, kFull};
        }
        if (b == nb_) return;
        u64 nl = 0, nt = 0;
        for (std::size_t i = lo_of(b), e = hi_of(b); i < e && cum < need; ++i) {
            if (top_[i] > p) {
                cum += trail_gain(m_[i], p);
                ++nt;
            } else {
                if (top_[i] == p) cum += lead_gain(m_[i], p);
                ++nl;
            }
        }
        st[b] = {nl, nt};
        return;
    }
    auto scan = [&](bool lead, double left) {
        double cum = 0;
        std::size_t b = 0;
        for (; b < nb_; ++b) {
            const double br = lead ? per[b].red_lead : per[b].red_trail;
            if (cum + br >= left) break;
            cum += br;
            (lead ? st[b].lead : st[b].trail) = kFull;
        }
        if (b == nb_) return;
        u64 c = 0;
        for (std::size_t i = lo_of(b), e = hi_of(b); i < e && cum < left; ++i) {
            if (lead) {
                if (top_[i] > p) continue;
                if (top_[i] == p) cum += lead_gain(m_[i], p);
            } else {
                if (top_[i] <= p) continue;
                cum += trail_gain(m_[i], p);
            }
            ++c;
        }
        (lead ? st[b].lead : st[b].trail) = c;
    };
    const double first = lead_first ? tot.red_lead : tot.red_trail;
    if (first >= need) {
        scan(lead_first, need);
        return;
    }
    for (auto& s : st) (lead_first ? s.lead : s.trail) = kFull;
    scan(!lead_first, need - first);
}

// Decoder-side magnitudes implied by the plan (core_codec.cpp:344-367).
void CoreEncoder::decode_model() {
    const int lp = plan_.last_plane;
    plan_.decoded.assign(m_.size(), 0);
    for (std::size_t b = 0; b < nb_; ++b) {
        u64 nl = 0, nt = 0;
        for (std::size_t i = lo_of(b), e = hi_of(b); i < e; ++i) {
            int pe;
            if (top_[i] > lp) {
                pe = (nt++ < plan_.stops[b].trail) ? lp : lp + 1;
            } else {
                const bool inside = nl++ < plan_.stops[b].lead;
                if (top_[i] != lp || !inside) continue;
                pe = lp;
            }
            u64 v = (m_[i] >> pe) << pe;
            if (pe >= 1) v += u64{1} << (pe - 1);
            plan_.decoded[i] = v;
        }
    }
}

Stream CoreEncoder::finalize(std::span<const u8> neg) {
    if (!done_) throw Error("core codec: finalize before plan");
    if (neg.size() != m_.size()) throw Error("core codec: sign count mismatch");
    Stream s;
    s.last_plane = plan_.last_plane;
    s.block = bs_;
    s.stops = plan_.stops;
    s.payloads.resize(plan_.n_planes);
    for (int rel = 0; rel < plan_.n_planes; ++rel) {
        const int p = 63 - rel;
        s.payloads[rel].resize(nb_);
        for (std::size_t b = 0; b < nb_; ++b) {
            const bool bp = p == plan_.last_plane;
            s.payloads[rel][b] = emit(p, b, bp ? plan_.stops[b].lead : kFull,
                                      bp ? plan_.stops[b].trail : kFull, neg.data(), nullptr);
        }
    }
    double sse = 0;
    for (std::size_t i = m_.size(); i-- > 0;) {
        const double r = dbl(m_[i]) - dbl(plan_.decoded[i]);
        sse += r * r;
    }
    s.achieved_int = sse;
    return s;
}

// ---------------------------------------------------------------- decoder
namespace {
u32 le32(std::span<const u8> in, std::size_t pos) {
    if (pos + 4 > in.size()) throw Error("core codec: truncated block payload");
    u32 v = 0;
    for (int i = 0; i < 4; ++i) v |= static_cast<u32>(in[pos + i]) << (8 * i);
    return v;
}
}  // namespace

Decoded decode_stream(const StreamMeta& meta, const std::vector<std::vector<std::span<const u8>>>& pl) {
    const u64 n = meta.count, bs = meta.block;
    if (bs == 0 && n > 0) throw Error("core decode: zero block size");
    const std::size_t nb = n == 0 ? 0 : (n + bs - 1) / bs;
    if (meta.stops.size() != nb) throw Error("core decode: stop table size mismatch");
    for (const auto& row : pl)
        if (row.size() != nb) throw Error("core decode: payload block count mismatch");
    const std::size_t planes = pl.size();
    if (planes != static_cast<std::size_t>(64 - meta.last_plane) && !(planes == 0 && meta.last_plane == 63))
        throw Error("core decode: plane count does not match last plane");
    Decoded d;
    d.mag.assign(n, 0);
    d.neg.assign(n, 0);
    std::vector<u8> pe(n, 0);
    for (std::size_t b = 0; b < nb; ++b) {
        const std::size_t lo = b * bs, hi = std::min<std::size_t>(lo + bs, n);
        for (std::size_t rel = 0; rel < planes; ++rel) {
            const int p = 63 - static_cast<int>(rel);
            const bool last = p == meta.last_plane;
            const u64 ls = last ? meta.stops[b].lead : kFull;
            const u64 ts = last ? meta.stops[b].trail : kFull;
            const auto pay = pl[rel][b];
            const u32 elen = le32(pay, 0);
            if (4 + static_cast<std::size_t>(elen) > pay.size())
                throw Error("core decode: entropy section overruns payload");
            u64 insig = 0;
            for (std::size_t i = lo; i < hi; ++i) insig += d.mag[i] == 0;
            const u64 clen = std::min<u64>(insig, ls);
            std::vector<u8> col;
            if (clen > 0) {
                if (elen == 0) throw Error("core decode: missing leading column");
                const auto runs = unpack_symbols(pay.subspan(4, elen));
                for (std::size_t r = 0; r + 1 < runs.size(); ++r) {
                    col.insert(col.end(), runs[r], 0);
                    col.push_back(1);
                }
                col.insert(col.end(), runs.back(), 0);
                if (col.size() != clen) throw Error("rle: run lengths do not match column length");
            }
            const auto raw = pay.subspan(4 + elen);
            std::size_t rb = 0;
            auto rd = [&]() {
                if ((rb >> 3) >= raw.size()) throw Error("bit reader: read past end");
                const bool v = (raw[rb >> 3] >> (7 - (rb & 7))) & 1u;
                ++rb;
                return v;
            };
            u64 lu = 0, tu = 0, cp = 0;
            for (std::size_t i = lo; i < hi; ++i) {
                if (d.mag[i] != 0) {
                    if (tu < ts) {
                        if (rd()) d.mag[i] |= u64{1} << p;
                        pe[i] = static_cast<u8>(p);
                        ++tu;
                    }
                } else if (lu < ls && cp < col.size()) {
                    const bool one = col[cp++] != 0;
                    ++lu;
                    if (one) {
                        d.mag[i] = u64{1} << p;
                        d.neg[i] = rd() ? 1 : 0;
                        pe[i] = static_cast<u8>(p);
                    }
                }
            }
        }
        for (std::size_t i = lo; i < hi; ++i)
            if (d.mag[i] != 0 && pe[i] >= 1) d.mag[i] += u64{1} << (pe[i] - 1);
    }
    return d;
}

std::vector<std::vector<u8>> dead_slices(const Shape& shape, std::span<const u64> dec, std::span<const u64> order) {
    std::vector<std::vector<u8>> dead(shape.size());
    for (std::size_t a = 0; a < shape.size(); ++a) dead[a].assign(shape[a], 1);
    const auto st = strides_of(shape);
    for (std::size_t v = 0; v < dec.size(); ++v) {
        if (!dec[v]) continue;
        const u64 pos = order.empty() ? v : order[v];
        for (std::size_t a = 0; a < shape.size(); ++a) dead[a][(pos / st[a]) % shape[a]] = 0;
    }
    return dead;
}

}  // namespace orc
