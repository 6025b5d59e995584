// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp).
// Restates /root/reference/proj/src/entropy.cpp: MSB-first bit packing
// (:22-33), zero-run extraction (:51-64), the 32-bit-range / 64-bit-low range
// coder with LZMA-style carry (:82-118), the adaptive escape model (:155-239),
// the semi-static rANS backend (:290-388) and the symbol framing (:429-468).
#include <algorithm>
#include <map>
#include <unordered_map>

#include "orc.hpp"

namespace orc {

void BitSink::put(bool b) {
    if ((nbits_ & 7) == 0) buf_.push_back(0);
    if (b) buf_.back() |= static_cast<u8>(0x80u >> (nbits_ & 7));
    ++nbits_;
}

std::vector<u64> zero_runs(const std::vector<u8>& column) {
    std::vector<u64> runs;
    u64 zeros = 0;
    for (u8 bit : column) {
        if (bit) {
            runs.push_back(zeros);
            zeros = 0;
        } else {
            ++zeros;
        }
    }
    runs.push_back(zeros);  // trailing zeros, possibly the whole column
    return runs;
}

namespace {

// ---- range coder (entropy.cpp:82-118) ----
struct RangeCoder {
    Bytes& out;
    u64 low = 0;
    u32 range = 0xFFFFFFFFu;
    u8 cache = 0;
    u64 pending = 1;

    explicit RangeCoder(Bytes& o) : out(o) {}

    void shift() {
        const bool settle = static_cast<u32>(low) < 0xFF000000u || (low >> 32) != 0;
        if (settle) {
            const u8 carry = static_cast<u8>(low >> 32);
            u8 first = cache;
            while (pending) {
                out.push_back(static_cast<u8>(first + carry));
                first = 0xFF;
                --pending;
            }
            cache = static_cast<u8>(low >> 24);
        }
        ++pending;
        low = (low << 8) & 0xFFFFFFFFull;
    }
    void code(u32 cum, u32 freq, u32 total) {
        range /= total;
        low += static_cast<u64>(cum) * range;
        range *= freq;
        while (range < (1u << 24)) {
            shift();
            range <<= 8;
        }
    }
    void raw32(u64 v) {
        for (int i = 31; i >= 0; --i) code(static_cast<u32>((v >> i) & 1u), 1, 2);
    }
    void finish() {
        for (int i = 0; i < 5; ++i) shift();
    }
};

struct RangeReader {
    std::span<const u8> in;
    std::size_t pos = 0;
    u32 range = 0xFFFFFFFFu, code = 0;
    explicit RangeReader(std::span<const u8> s) : in(s) {
        for (int i = 0; i < 5; ++i) code = (code << 8) | next();
    }
    u8 next() { return pos < in.size() ? in[pos++] : 0; }
    u32 target(u32 total) {
        range /= total;
        const u32 t = code / range;
        return t >= total ? total - 1 : t;
    }
    void consume(u32 cum, u32 freq) {
        code -= cum * range;
        range *= freq;
        while (range < (1u << 24)) {
            code = (code << 8) | next();
            range <<= 8;
        }
    }
    u64 raw32() {
        u64 v = 0;
        for (int i = 0; i < 32; ++i) {
            const u32 t = target(2);
            consume(t, 1);
            v = (v << 1) | t;
        }
        return v;
    }
};

// ---- adaptive model (entropy.cpp:155-239) ----
// Index 0 is the escape.  Counts start at 1 (escape) / 32 (new symbol), grow by
// 32 per hit, and every count halves (floor, min 1) when total+32 would reach
// 2^16.  prefix(i) = sum of counts below index i; any exact prefix structure
// reproduces the reference's Fenwick tree values.
struct Model {
    std::vector<u64> sym{0};
    std::vector<u32> cnt{1};
    std::vector<u32> tree;  // Fenwick over cnt, 1-based
    std::unordered_map<u64, u32> index;
    u32 total = 1;

    Model() { rebuild(); }
    void rebuild() {
        std::size_t cap = 2;
        while (cap < cnt.size() + 1) cap *= 2;
        tree.assign(cap, 0);
        for (u32 i = 0; i < cnt.size(); ++i) add(i, cnt[i]);
    }
    void add(u32 i, u32 d) {
        for (std::size_t j = i + 1; j < tree.size(); j += j & (~j + 1)) tree[j] += d;
    }
    u32 below(u32 i) const {
        u32 s = 0;
        for (std::size_t j = i; j > 0; j -= j & (~j + 1)) s += tree[j];
        return s;
    }
    u32 locate(u32 target) const {  // index whose interval holds target
        u32 lo = 0, hi = static_cast<u32>(cnt.size()) - 1;
        while (lo < hi) {  // largest i with below(i) <= target
            const u32 mid = (lo + hi + 1) / 2;
            if (below(mid) <= target) lo = mid; else hi = mid - 1;
        }
        return lo;
    }
    void halve() {
        total = 0;
        for (auto& c : cnt) {
            c = std::max<u32>(1, c >> 1);
            total += c;
        }
        rebuild();
    }
    void hit(u32 i) {
        if (total + 32 >= (1u << 16)) halve();
        cnt[i] += 32;
        total += 32;
        add(i, 32);
    }
    void fresh(u64 s) {
        if (total + 32 >= (1u << 16)) halve();
        const u32 i = static_cast<u32>(cnt.size());
        sym.push_back(s);
        cnt.push_back(32);
        if (cnt.size() + 1 > tree.size()) rebuild();
        else add(i, 32);
        total += 32;
        index.emplace(s, i);
    }
    void put(RangeCoder& rc, u64 s) {
        auto it = index.find(s);
        if (it != index.end()) {
            rc.code(below(it->second), cnt[it->second], total);
            hit(it->second);
            return;
        }
        rc.code(0, cnt[0], total);
        if (s > 0xFFFFFFFFull) throw Error("entropy: run length exceeds 32 bits");
        rc.raw32(s);
        fresh(s);
    }
    u64 get(RangeReader& rr) {
        const u32 t = rr.target(total);
        const u32 i = locate(t);
        rr.consume(below(i), cnt[i]);
        if (i == 0) {
            const u64 s = rr.raw32();
            fresh(s);
            return s;
        }
        const u64 s = sym[i];
        hit(i);
        return s;
    }
};

// ---- semi-static rANS (entropy.cpp:290-421) ----
void varint(Bytes& o, u64 v) {
    for (; v >= 0x80; v >>= 7) o.push_back(static_cast<u8>(v) | 0x80u);
    o.push_back(static_cast<u8>(v));
}
u64 read_varint(std::span<const u8> in, std::size_t& pos) {
    u64 v = 0;
    for (unsigned sh = 0;; sh += 7) {
        if (pos >= in.size()) throw Error("entropy: truncated varint");
        const u8 b = in[pos++];
        v |= static_cast<u64>(b & 0x7F) << sh;
        if (!(b & 0x80)) return v;
        if (sh + 7 > 63) throw Error("entropy: varint overflow");
    }
}

struct Table {
    u32 bits = 12;
    std::vector<u64> sym;
    std::vector<u32> f, c;
};

Table make_table(std::span<const u64> s) {
    std::map<u64, u64> h;
    for (u64 v : s) ++h[v];
    Table t;
    while ((u64{1} << t.bits) < h.size()) ++t.bits;
    const u64 scale = u64{1} << t.bits;
    u64 sum = 0;
    for (auto [v, n] : h) {
        u64 q = n * scale / s.size();
        if (q == 0) q = 1;
        t.sym.push_back(v);
        t.f.push_back(static_cast<u32>(q));
        sum += q;
    }
    while (sum != scale) {
        const bool grow = sum < scale;
        std::size_t pick = 0;
        for (std::size_t i = 1; i < t.f.size(); ++i) {
            const bool better = grow ? t.f[i] > t.f[pick] : (t.f[i] > t.f[pick] && t.f[i] > 1);
            if (better) pick = i;
        }
        if (grow) {
            ++t.f[pick];
            ++sum;
        } else {
            if (t.f[pick] <= 1) throw Error("entropy: cannot normalize rans table");
            --t.f[pick];
            --sum;
        }
    }
    t.c.assign(t.f.size() + 1, 0);
    for (std::size_t i = 0; i < t.f.size(); ++i) t.c[i + 1] = t.c[i] + t.f[i];
    return t;
}

void rans_put(Bytes& o, std::span<const u64> s) {
    const Table t = make_table(s);
    varint(o, t.sym.size());
    varint(o, t.bits);
    u64 prev = 0;
    for (std::size_t i = 0; i < t.sym.size(); ++i) {
        varint(o, t.sym[i] - prev);
        varint(o, t.f[i]);
        prev = t.sym[i];
    }
    constexpr u64 L = u64{1} << 31;
    u64 x = L;
    std::vector<u32> words;
    for (std::size_t i = s.size(); i-- > 0;) {
        const std::size_t j = static_cast<std::size_t>(
            std::lower_bound(t.sym.begin(), t.sym.end(), s[i]) - t.sym.begin());
        const u64 f = t.f[j];
        const u64 lim = ((L >> t.bits) << 32) * f;
        while (x >= lim) {
            words.push_back(static_cast<u32>(x));
            x >>= 32;
        }
        x = ((x / f) << t.bits) + (x % f) + t.c[j];
    }
    for (int i = 0; i < 8; ++i) o.push_back(static_cast<u8>(x >> (8 * i)));
    for (std::size_t w = words.size(); w-- > 0;)
        for (int b = 0; b < 4; ++b) o.push_back(static_cast<u8>(words[w] >> (8 * b)));
}

void rans_get(std::span<const u8> in, std::size_t count, std::vector<u64>& out) {
    std::size_t pos = 0;
    Table t;
    const u64 n = read_varint(in, pos);
    t.bits = static_cast<u32>(read_varint(in, pos));
    if (t.bits > 20) throw Error("entropy: bad rans table");
    u64 prev = 0, total = 0;
    for (u64 i = 0; i < n; ++i) {
        prev += read_varint(in, pos);
        t.sym.push_back(prev);
        t.f.push_back(static_cast<u32>(read_varint(in, pos)));
        total += t.f.back();
    }
    if (n > 0 && total != (u64{1} << t.bits)) throw Error("entropy: bad rans table total");
    t.c.assign(n + 1, 0);
    for (std::size_t i = 0; i < n; ++i) t.c[i + 1] = t.c[i] + t.f[i];
    if (count > 0 && n == 0) throw Error("entropy: empty rans table");
    if (pos + 8 > in.size()) throw Error("entropy: truncated rans payload");
    u64 x = 0;
    for (int i = 0; i < 8; ++i) x |= static_cast<u64>(in[pos + i]) << (8 * i);
    pos += 8;
    const u64 mask = (u64{1} << t.bits) - 1;
    for (std::size_t i = 0; i < count; ++i) {
        const u32 slot = static_cast<u32>(x & mask);
        const std::size_t j = static_cast<std::size_t>(
            std::upper_bound(t.c.begin(), t.c.end(), slot) - t.c.begin()) - 1;
        if (j >= n) throw Error("entropy: corrupt rans payload");
        out.push_back(t.sym[j]);
        x = t.f[j] * (x >> t.bits) + slot - t.c[j];
        while (x < (u64{1} << 31)) {
            if (pos + 4 > in.size()) throw Error("entropy: truncated rans payload");
            u32 w = 0;
            for (int b = 0; b < 4; ++b) w |= static_cast<u32>(in[pos + b]) << (8 * b);
            pos += 4;
            x = (x << 32) | w;
        }
    }
}

}  // namespace

Bytes pack_symbols(Coder c, std::span<const u64> syms) {
    if (syms.size() > 0xFFFFFFFFull) throw Error("entropy: too many symbols");
    Bytes o;
    o.push_back(static_cast<u8>(c));
    const u32 n = static_cast<u32>(syms.size());
    for (int i = 0; i < 4; ++i) o.push_back(static_cast<u8>(n >> (8 * i)));
    if (syms.empty()) return o;
    if (c == Coder::ac) {
        RangeCoder rc(o);
        Model m;
        for (u64 s : syms) m.put(rc, s);
        rc.finish();
    } else {
        rans_put(o, syms);
    }
    return o;
}

std::vector<u64> unpack_symbols(std::span<const u8> p) {
    if (p.size() < 5) throw Error("entropy: truncated payload");
    u32 n = 0;
    for (int i = 0; i < 4; ++i) n |= static_cast<u32>(p[1 + i]) << (8 * i);
    std::vector<u64> out;
    out.reserve(n);
    if (n == 0) return out;
    const auto body = p.subspan(5);
    if (p[0] == static_cast<u8>(Coder::ac)) {
        RangeReader rr(body);
        Model m;
        for (u32 i = 0; i < n; ++i) out.push_back(m.get(rr));
    } else if (p[0] == static_cast<u8>(Coder::rans)) {
        rans_get(body, n, out);
    } else {
        throw Error("entropy: unknown coder id");
    }
    return out;
}

}  // namespace orc
