// Device decompress: pipeline::decompress / decompress_tensor
// (pipeline.cpp:197-236, 266-283).  The host parses the container (container.cpp
// read_container layout; error texts as the reference) and builds one
// descriptor per (stream, plane, block) payload; the device decodes every
// entropy section at once, rebuilds all streams block-parallel, expands the
// factors from their reflectors, dequantises the core and applies the factors
// in the decompression mode order (sthosvd.cpp:35-63, 173-218) with the DMMA
// TTM kernel, then casts to the source dtype (container.cpp:98-140).
#include "decompress.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>

#include "decode.cuh"
#include "kernels.cuh"
#include "pipeline.hpp"
#include "quant.cuh"

namespace tcb {

namespace {

struct Rd {
    const u8* b;
    u64 n;
    u64 pos = 0;
    std::string sec;
    void need(u64 k) const {
        if (pos + k > n) throw Error("container: truncated " + sec + " section");
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
    u64 skip(u64 k) {  // returns the absolute offset of the skipped span
        need(k);
        const u64 at = pos;
        pos += k;
        return at;
    }
};

struct StreamParse {
    u64 count = 0, block = 0;
    int last_plane = 63;
    u32 nb = 0, np = 0;
    std::vector<u64> lead, trail;
    std::vector<std::pair<u64, u64>> pay;  // (absolute offset, length), plane-major
};

StreamParse get_stream(Rd& r, u64 base) {
    StreamParse v;
    v.count = r.u64v();
    v.block = r.u64v();
    v.last_plane = r.u8v();
    v.nb = r.u32v();
    v.lead.resize(v.nb);
    v.trail.resize(v.nb);
    for (u32 b = 0; b < v.nb; ++b) {
        v.lead[b] = r.u64v();
        v.trail[b] = r.u64v();
    }
    v.np = r.u32v();
    if (v.np > 64) throw Error("container: implausible plane count");
    for (u32 p = 0; p < v.np; ++p)
        for (u32 b = 0; b < v.nb; ++b) {
            const u32 len = r.u32v();
            const u64 at = r.skip(len);
            v.pay.push_back({base + at, len});
        }
    return v;
}

// exhaustive minimum of sum_i n_{q1}..n_{qi} r_{qi}..r_{qd} (sthosvd.cpp:35-63)
std::vector<u64> decompression_order(const std::vector<u64>& n, const std::vector<u64>& r) {
    const std::size_t d = n.size();
    if (d > 8) throw Error("mode order: exhaustive search limited to order 8");
    std::vector<u64> perm(d);
    for (std::size_t i = 0; i < d; ++i) perm[i] = i;
    auto cost = [&](const std::vector<u64>& q) {
        unsigned __int128 tot = 0;
        for (std::size_t i = 0; i < d; ++i) {
            unsigned __int128 t = 1;
            for (std::size_t j = 0; j <= i; ++j) t *= n[q[j]];
            for (std::size_t j = i; j < d; ++j) t *= r[q[j]];
            tot += t;
        }
        return tot;
    };
    std::vector<u64> best = perm;
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

std::vector<u64> inverse(const std::vector<u64>& p) {
    std::vector<u64> q(p.size());
    for (std::size_t i = 0; i < p.size(); ++i) q[p[i]] = i;
    return q;
}

u64 prod(const std::vector<u64>& v) {
    u64 t = 1;
    for (auto x : v) t *= x;
    return t;
}

u64 le32(const u8* p) {
    return static_cast<u64>(p[0]) | (static_cast<u64>(p[1]) << 8) | (static_cast<u64>(p[2]) << 16) |
           (static_cast<u64>(p[3]) << 24);
}

const char* dec_message(int e) {
    switch (e) {
        case kDecErrEntropy: return "entropy: corrupt payload";
        case kDecErrCoder: return "entropy: unknown coder id";
        case kDecErrModel: return "entropy: model capacity exceeded";
        case kDecErrMissingColumn: return "core decode: missing leading column";
        case kDecErrRle: return "rle: run lengths do not match column length";
        case kDecErrBits: return "bit reader: read past end";
        default: return "core decode: corrupt stream";
    }
}

struct FactorMeta {
    std::vector<u8> dead;
    std::vector<double> sn;
    int k = 0;
    u64 count = 0;
};

}  // namespace

ContainerHeader parse_header(const u8* c, u64 len, u64* end) {
    Rd r{c, len, 0, "header"};
    if (len < 4 || std::memcmp(c, "TKC1", 4) != 0) throw Error("container: bad magic");
    r.pos = 4;
    ContainerHeader h;
    h.version = r.u8v();
    if (h.version != 1) throw Error("container: unsupported format version " + std::to_string(h.version));
    h.dtype = r.u8v();
    if (h.dtype > 9) throw Error("container: unknown source dtype");
    h.f32 = r.u8v() != 0;
    const std::size_t d = r.u8v();
    if (d == 0) throw Error("container: zero tensor order");
    h.coder = r.u8v();  // each entropy section carries its own id too
    if (h.coder > 1) throw Error("container: unknown entropy coder id");
    h.method = r.u8v();
    if (h.method > 2) throw Error("container: unknown vectorization method id");
    const u8 flags = r.u8v();
    h.zero = flags & 1;
    h.split = flags & 2;
    h.simple = flags & 4;
    r.u8v();
    h.n.resize(d);
    h.rk.resize(d);
    h.order.resize(d);
    h.storage.resize(d);
    for (auto& v : h.n) v = r.u64v();
    for (auto& v : h.rk) v = r.u64v();
    for (auto& v : h.order) v = r.u8v();
    for (auto& v : h.storage) v = r.u8v();
    auto is_perm = [&](const std::vector<u64>& p) {
        std::vector<u8> seen(d, 0);
        for (auto v : p) {
            if (v >= d || seen[v]) return false;
            seen[v] = 1;
        }
        return true;
    };
    if (!is_perm(h.order) || !is_perm(h.storage)) throw Error("container: corrupt mode permutations");
    for (std::size_t i = 0; i < d; ++i)
        if (h.n[i] == 0 || h.rk[i] == 0 || h.rk[i] > h.n[i]) throw Error("container: corrupt mode sizes or ranks");
    h.k = static_cast<std::int32_t>(r.u32v());
    h.block = r.u64v();
    h.rtmss = r.f64v();
    h.target_sse = r.f64v();
    h.norm_sq = r.f64v();
    h.trunc_sse = r.f64v();
    h.cq_sse = r.f64v();
    h.est_sse = r.f64v();
    *end = r.pos;
    return h;
}

namespace {

struct Sections {
    std::vector<FactorMeta> fm;
    std::vector<StreamParse> sp;  // factor streams, then the core stream
};

// factor and core sections (container.cpp read_container's section loop)
Sections parse_sections(const u8* c, u64 len, u64 pos, const ContainerHeader& h) {
    Rd r{c, len, pos, "header"};
    const std::size_t d = h.n.size();
    Sections o;
    o.fm.resize(d);
    for (std::size_t i = 0; i < d; ++i) {
        const u64 flen = r.u64v();
        const u64 at = r.skip(flen);
        Rd fr{c + at, flen, 0, "factor " + std::to_string(i + 1)};
        auto& f = o.fm[i];
        f.dead.assign(h.rk[i], 0);
        for (u64 j = 0; j < h.rk[i]; j += 8) {
            const u8 b = fr.u8v();
            for (u64 q = 0; q < 8 && j + q < h.rk[i]; ++q) f.dead[j + q] = (b >> q) & 1;
        }
        f.sn.resize(h.rk[i]);
        for (auto& v : f.sn) v = fr.f64v();
        f.k = static_cast<std::int32_t>(fr.u32v());
        f.count = fr.u64v();
        o.sp.push_back(get_stream(fr, at));
        if (o.sp.back().count != f.count) throw Error("container: factor stream length mismatch");
    }
    {
        const u64 clen = r.u64v();
        const u64 at = r.skip(clen);
        Rd cr{c + at, clen, 0, "core"};
        o.sp.push_back(get_stream(cr, at));
    }
    std::vector<u64> cp(d), cs(d);
    for (std::size_t j = 0; j < d; ++j) cp[j] = h.rk[h.order[j]];
    for (std::size_t a = 0; a < d; ++a) cs[a] = cp[h.storage[a]];
    if (o.sp.back().count != prod(cs)) throw Error("container: core length does not match ranks");
    return o;
}

}  // namespace

ContainerHeader read_container_header(const u8* c, u64 len) {
    u64 pos = 0;
    ContainerHeader h = parse_header(c, len, &pos);
    if (!h.zero) parse_sections(c, len, pos, h);
    return h;
}

DecompressOut decompress_device(const u8* c, u64 len, cudaStream_t s) {
    const auto t0 = std::chrono::steady_clock::now();
    HostTrace ht("decompress: parse");
    u64 hpos = 0;
    const ContainerHeader h = parse_header(c, len, &hpos);
    DecompressOut out;
    out.dtype = h.dtype;
    out.f32 = h.f32;
    const std::size_t d = h.n.size();
    const bool zero = h.zero, simple = h.simple;
    const int method = h.method;
    const int k = h.k;
    const auto& n = h.n;
    const auto& rk = h.rk;
    const auto& order = h.order;
    const auto& storage = h.storage;
    out.shape = n;
    const u64 total = prod(n);
    out.x = DevBuf<double>(total, s);
    if (zero) {
        TCB_CUDA(cudaMemsetAsync(out.x.p, 0, total * sizeof(double), s));
        out.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        return out;
    }
    Sections secs = parse_sections(c, len, hpos, h);
    auto& fm = secs.fm;
    auto& sp = secs.sp;
    std::vector<u64> cp(d), cs(d);
    for (std::size_t j = 0; j < d; ++j) cp[j] = rk[order[j]];
    for (std::size_t a = 0; a < d; ++a) cs[a] = cp[storage[a]];
    // ---- descriptors (decode_stream's checks, core_codec.cpp:421-440)
    std::vector<DecSection> sec;
    std::vector<DecStream> ds(sp.size());
    std::vector<DecBlock> blk;
    std::vector<u64> stops;  // lead | trail per stream, concatenated
    u64 nsym_tot = 0, scratch_tot = 0, coef_tot = 0;
    for (std::size_t si = 0; si < sp.size(); ++si) {
        const auto& v = sp[si];
        if (v.block == 0 && v.count > 0) throw Error("core decode: zero block size");
        const u64 nb = v.count == 0 ? 0 : (v.count + v.block - 1) / v.block;
        if (v.nb != nb) throw Error("core decode: stop table size mismatch");
        if (v.np != static_cast<u32>(64 - v.last_plane) && !(v.np == 0 && v.last_plane == 63))
            throw Error("core decode: plane count does not match last plane");
        DecStream& st = ds[si];
        st.count = v.count;
        st.block = v.block;
        st.last_plane = v.last_plane;
        st.nb = v.nb;
        st.nplanes = v.np;
        st.sec_off = sec.size();
        st.out_off = coef_tot;
        coef_tot += v.count;
        for (const auto& [at, plen] : v.pay) {
            DecSection e;
            if (plen < 4) throw Error("container: truncated core section");
            e.elen = static_cast<u32>(le32(c + at));
            if (4 + static_cast<u64>(e.elen) > plen) throw Error("core decode: entropy section overruns payload");
            e.ent_off = at + 4;
            e.ent_len = e.elen;
            e.raw_off = at + 4 + e.elen;
            e.raw_len = plen - 4 - e.elen;
            if (e.elen > 0) {
                if (e.elen < 5) throw Error("entropy: truncated payload");
                e.nsym = static_cast<u32>(le32(c + at + 5));
                e.cap = (e.nsym + 2) & ~1u;
                e.sym_off = nsym_tot;
                nsym_tot += e.nsym;
                const u8 coder = c[at + 4];
                if (coder == 1) {  // rANS table: u64 symbols first, so keep 8-byte alignment
                    e.scratch_off = (scratch_tot + 1) & ~u64{1};
                    scratch_tot = e.scratch_off + 5ull * e.nsym + 4;
                } else if (e.cap > 2048) {
                    e.scratch_off = (scratch_tot + 1) & ~u64{1};
                    scratch_tot = e.scratch_off + decode_model_words(e.cap);
                }
            }
            sec.push_back(e);
        }
        for (u32 b = 0; b < nb; ++b) {
            DecBlock bk;
            bk.stream = static_cast<u32>(si);
            bk.b = b;
            bk.lo = static_cast<u64>(b) * v.block;
            bk.hi = std::min(v.count, bk.lo + v.block);
            blk.push_back(bk);
        }
        stops.insert(stops.end(), v.lead.begin(), v.lead.end());
        stops.insert(stops.end(), v.trail.begin(), v.trail.end());
    }
    ht.stop();
    HostTrace ht_dev("decompress: entropy+streams");
    // ---- device
    DevBuf<u8> dc(len, s);
    dc.upload(c, len);
    DevBuf<u64> dstops(std::max<u64>(stops.size(), 1), s);
    if (!stops.empty()) dstops.upload(stops.data(), stops.size());
    {
        u64 so = 0;
        for (std::size_t si = 0; si < sp.size(); ++si) {
            ds[si].stops_lead = dstops.p + so;
            ds[si].stops_trail = dstops.p + so + sp[si].nb;
            so += 2ull * sp[si].nb;
        }
    }
    DevBuf<DecSection> dsec(std::max<std::size_t>(sec.size(), 1), s);
    if (!sec.empty()) dsec.upload(sec.data(), sec.size());
    DevBuf<DecStream> dstr(ds.size(), s);
    dstr.upload(ds.data(), ds.size());
    DevBuf<DecBlock> dblk(std::max<std::size_t>(blk.size(), 1), s);
    if (!blk.empty()) dblk.upload(blk.data(), blk.size());
    DevBuf<u64> syms(std::max<u64>(nsym_tot, 1), s);
    DevBuf<u32> scratch(std::max<u64>(scratch_tot, 2), s);
    DevBuf<u64> mag(std::max<u64>(coef_tot, 1), s);
    DevBuf<u8> neg(std::max<u64>(coef_tot, 1), s), pe(std::max<u64>(coef_tot, 1), s),
        colb(std::max<u64>(coef_tot, 1), s);
    DevBuf<int> err(1, s);
    err.zero();
    decode_entropy(dc.p, dsec.p, sec, syms.p, scratch.p, err.p, s);
    decode_streams(dc.p, dstr.p, dblk.p, blk.size(), dsec.p, syms.p, mag.p, neg.p, pe.p, colb.p, err.p, s);
    // no host round trip here: the factor and reconstruction launches below are
    // enqueued while the decode kernels run (their sizes come from the parsed
    // header, so a corrupt stream only yields garbage values, never an out-of-range
    // access); both error flags are read once at the end, the decode one first
    ht_dev.stop();
    HostTrace ht_rec("decompress: factors+reconstruct");
    // ---- factors (decode_factor, factor_codec.cpp:246-264): independent, each on its
    // own side stream (small launches that overlap), one shared error flag
    std::vector<DevBuf<double>> U(d);
    DevBuf<int> ferr(1, s);
    ferr.zero();
    static PerDevice<std::vector<cudaStream_t>> side_dev;
    const std::vector<cudaStream_t>& side = side_dev.get([] {
        std::vector<cudaStream_t> v(8);
        for (auto& st : v) TCB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        return v;
    });
    for (std::size_t i = 0; i < d; ++i) U[i] = DevBuf<double>(n[i] * rk[i], s);
    cudaEvent_t fork_ev, join_ev[8];
    TCB_CUDA(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    TCB_CUDA(cudaEventRecord(fork_ev, s));
    for (std::size_t i = 0; i < d; ++i) {
        cudaStream_t si = side[i % side.size()];
        TCB_CUDA(cudaStreamWaitEvent(si, fork_ev, 0));
        const auto& f = fm[i];
        std::vector<u64> live;
        std::vector<double> ln;
        for (u64 j = 0; j < rk[i]; ++j)
            if (!f.dead[j]) {
                live.push_back(j);
                ln.push_back(f.sn[j]);
            }
        const u64 rl = live.size();
        if (rl > 0 && f.count != n[i] * rl - rl * (rl + 1) / 2)
            throw Error("factor decode: coefficient count mismatch");
        std::vector<double> sc(rl);
        if (rl > 0) {
            if (simple) {
                sc = ln;
            } else {
                const auto al = alpha_weights(ln, n[i]);
                for (u64 j = 0; j < rl; ++j) sc[j] = std::sqrt(2.0 * al[j]);
            }
        }
        DevBuf<double> dsc(std::max<u64>(rl, 1), si);
        if (rl > 0) dsc.upload(sc.data(), rl);
        factor_expand(mag.p + ds[i].out_off, neg.p + ds[i].out_off, f.k, n[i], rk[i], live, dsc.p, U[i].p, si,
                      ferr.p);
        if (i < 8) {
            TCB_CUDA(cudaEventCreateWithFlags(&join_ev[i], cudaEventDisableTiming));
            TCB_CUDA(cudaEventRecord(join_ev[i], si));
            TCB_CUDA(cudaStreamWaitEvent(s, join_ev[i], 0));
        }
    }
    cudaEventDestroy(fork_ev);
    for (std::size_t i = 0; i < d && i < 8; ++i) cudaEventDestroy(join_ev[i]);
    // ---- core: dequantise, storage -> processing order (pipeline.cpp:206-219)
    const u64 nc = prod(cs);
    DevBuf<double> core_s(nc, s), core_p(nc, s);
    const DevBuf<u64> vorder = order_map_device(method, cs, s);  // OrderMap::build (pipeline.cpp:210)
    dequantize(mag.p + ds[d].out_off, neg.p + ds[d].out_off, nc, k, core_s.p, s, vorder.p);
    permute_axes(core_s.p, core_p.p, cs, inverse(storage), s);
    core_s.release();
    // ---- reconstruct (sthosvd.cpp:173-218): decompression order, TTM expansions, final transpose
    const auto q = decompression_order(n, rk);
    const auto ip = inverse(order);
    std::vector<u64> ax(d);
    for (std::size_t j = 0; j < d; ++j) ax[j] = ip[q[j]];
    DevBuf<double> x(nc, s);
    permute_axes(core_p.p, x.p, cp, ax, s);
    core_p.release();
    std::vector<u64> cur(d);
    for (std::size_t j = 0; j < d; ++j) cur[j] = rk[q[j]];
    for (std::size_t step = 0; step < d; ++step) {
        const u64 mode = q[step];
        const u64 rows = cur[0], cols = prod(cur) / rows, nn = n[mode];
        DevBuf<double> ut(rows * nn, s);  // U^T: rows x nn
        permute_axes(U[mode].p, ut.p, std::vector<u64>{nn, rows}, std::vector<u64>{1, 0}, s);
        DevBuf<double> nx(cols * nn, s);
        ttm_f64(x.p, rows, cols, ut.p, nn, nx.p, s);
        x = std::move(nx);
        cur.erase(cur.begin());
        cur.push_back(nn);
    }
    permute_axes(x.p, out.x.p, cur, inverse(q), s);
    {
        int e = 0, fe = 0;
        err.download(&e, 1);
        ferr.download(&fe, 1);
        stream_sync(s);
        if (e) throw Error(dec_message(e));
        if (fe) throw Error("reconstruct: reflector sub-diagonal norm reaches 1");
    }
    out.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

u64 emit_size(const DecompressOut& t) {
    static const std::size_t sz[10] = {1, 1, 2, 2, 4, 4, 8, 8, 4, 8};
    return prod(t.shape) * sz[t.dtype];
}

void emit_bytes(const DecompressOut& t, u8* host, cudaStream_t s) {
    const u64 total = prod(t.shape), nb = emit_size(t);
    if (total == 0) return;
    if (t.dtype == 9) {  // fp64: the reconstruction itself
        TCB_CUDA(cudaMemcpyAsync(host, t.x.p, nb, cudaMemcpyDeviceToHost, s));
    } else {
        DevBuf<u8> db(nb, s);
        emit_dtype(t.x.p, total, t.dtype, db.p, s);
        TCB_CUDA(cudaMemcpyAsync(host, db.p, nb, cudaMemcpyDeviceToHost, s));
        stream_sync(s);
        return;
    }
    stream_sync(s);
}

std::vector<u8> emit_bytes(const DecompressOut& t, cudaStream_t s) {
    static const std::size_t sz[10] = {1, 1, 2, 2, 4, 4, 8, 8, 4, 8};
    const u64 total = prod(t.shape);
    std::vector<u8> bytes(total * sz[t.dtype]);
    if (total == 0) return bytes;
    DevBuf<u8> db(bytes.size(), s);
    emit_dtype(t.x.p, total, t.dtype, db.p, s);
    db.download(bytes.data(), bytes.size());
    stream_sync(s);
    return bytes;
}

}  // namespace tcb
