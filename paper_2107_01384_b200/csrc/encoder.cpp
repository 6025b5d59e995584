// Certified breakpoint logic for the device encoder.
//
// The reference decides the breakpoint plane, the recalibration points and the
// split-plane stops by comparing doubles it accumulates SERIALLY
// (core_codec.cpp:173-342, error_model.cpp:34-72).  The device computes every
// such sum exactly (double-double) together with a rigorous bound W on the
// serial rounding error (|fl_serial - exact| <= u * sum_k |partial_k| <= u*W),
// giving an interval that provably contains the reference's double.  Since
// round-to-nearest +,-,* and / by a positive constant are monotone, pushing
// both endpoints through the reference's own operation sequence yields an
// interval for every derived quantity; a comparison is certified when both
// endpoints agree.  Any uncertified comparison restarts planning in exact
// mode, where the device replays the sums serially in the reference's order.
//
// This TU must not be compiled with FMA contraction (host x86-64: no -mfma).
#include <cfloat>
#include <cmath>
#include <limits>

#include "encoder.hpp"

namespace tcb {

namespace {

struct Ambiguous {};

struct Iv {
    double lo, hi;
};
inline Iv pt(double x) { return {x, x}; }
inline Iv add(Iv a, Iv b) { return {a.lo + b.lo, a.hi + b.hi}; }
inline Iv sub(Iv a, Iv b) { return {a.lo - b.hi, a.hi - b.lo}; }

inline bool le(Iv a, Iv b) {  // a <= b
    if (a.hi <= b.lo) return true;
    if (a.lo > b.hi) return false;
    HostTrace ht("plan: ambiguous le");
    throw Ambiguous{};
}
inline bool ge(Iv a, Iv b) {  // a >= b
    if (a.lo >= b.hi) return true;
    if (a.hi < b.lo) return false;
    HostTrace ht("plan: ambiguous ge");
    throw Ambiguous{};
}

Iv from_sum(const SumRec& r, bool exact) {
    if (exact || r.nterms <= 1) return pt(r.hi + r.lo);  // serial replay, or 0/1 term: exact
    const double u = std::ldexp(1.0, -53);
    const double err = u * r.wabs * (1.0 + 1e-5) + std::ldexp(r.wabs, -70) + DBL_MIN;
    double lo = (r.hi - err) + r.lo;
    double hi = (r.hi + err) + r.lo;
    for (int i = 0; i < 2; ++i) {
        lo = std::nextafter(lo, -INFINITY);
        hi = std::nextafter(hi, INFINITY);
    }
    return {lo, hi};
}

struct Tot {
    Iv lead{0, 0}, trail{0, 0};
    u64 nlead = 0, nones = 0, ntrail = 0;
};

struct Planner {
    const u64* m;
    u64 n, block, nb;
    double target;
    EncodeOpts o;
    bool exact;
    cudaStream_t s;
    std::vector<PlaneBlockRec> batch;
    int batch_hi = -1, batch_lo = 64;

    // exact mode: every plane's serial statistics in one launch, and the initial
    // and every plane's recalibration sum in another (independent serial chains
    // side by side), computed on first use
    std::vector<PlaneBlockRec> ex_stats;
    std::vector<double> ex_sums;  // [0] initial, [1 + p] recalibration at plane p
    const PlaneBlockRec* stats(int p, int floor_p) {
        if (exact) {
            if (ex_stats.empty()) {
                HostTrace ht("plan: exact stats (all planes)");
                ex_stats.resize(nb * 64);
                plane_stats_serial_range(m, n, block, 63, 0, ex_stats.data(), s);
            }
            return ex_stats.data() + static_cast<u64>(63 - p) * nb;
        }
        if (p > batch_hi || p < batch_lo) {
            // planes per batch: every remaining plane when the core is small (each plane
            // is a pass over the magnitudes; one round trip instead of one per 8 planes)
            const int span = n <= (u64{1} << 18) ? 63 : n <= (u64{1} << 21) ? 15 : 7;
            const int lo = std::max(floor_p, p - span);
            batch.resize(nb * (p - lo + 1));
            HostTrace ht("plan: plane_stats batch");
            plane_stats(m, n, block, p, lo, batch.data(), s);
            batch_hi = p;
            batch_lo = lo;
        }
        return batch.data() + static_cast<u64>(batch_hi - p) * nb;
    }

    Iv block_sum(const SumRec& r) const { return from_sum(r, exact); }

    // crossing scan of one block, certified over the interval endpoints
    u64 cross(u64 b, int p, int cat, Iv cum, Iv need, u64* second = nullptr) {
        const double c[2] = {cum.lo, cum.hi};
        const double nd[2] = {need.hi, need.lo};
        u64 out[4];
        HostTrace ht("plan: crossing_scan");
        crossing_scan(m, n, block, b, p, cat, c, nd, 2, out, s);
        if (out[0] != out[2] || out[1] != out[3]) {
            HostTrace ht("plan: ambiguous crossing");
            throw Ambiguous{};
        }
        if (second) *second = out[1];
        return out[0];
    }

    void place_stops(int p, Iv need, const Tot& tot, const PlaneBlockRec* per, const Tot* prev, u64 prev_ebits,
                     std::vector<u64>& st) {
        bool lead_first = true;
        if (o.split && prev) {
            const double lc = static_cast<double>(prev_ebits + prev->nones);
            const double tc = static_cast<double>(prev->ntrail);
            auto eff = [](Iv red, double cost) -> Iv {
                if (cost > 0) return {red.lo / cost, red.hi / cost};
                if (red.lo > 0) return pt(HUGE_VAL);
                if (red.hi <= 0) return pt(0.0);
                throw Ambiguous{};
            };
            lead_first = ge(eff(prev->lead, lc), eff(prev->trail, tc));
        }
        if (!o.split) {
            Iv cum = pt(0.0);
            u64 b = 0;
            for (; b < nb; ++b) {
                const Iv br = add(block_sum(per[b].lead), block_sum(per[b].trail));
                if (ge(add(cum, br), need)) break;
                cum = add(cum, br);
                st[2 * b] = st[2 * b + 1] = kFull;
            }
            if (b == nb) return;
            u64 nt = 0;
            const u64 nl = cross(b, p, 2, cum, need, &nt);
            st[2 * b] = nl;
            st[2 * b + 1] = nt;
            return;
        }
        auto scan = [&](bool lead, Iv left) {
            Iv cum = pt(0.0);
            u64 b = 0;
            for (; b < nb; ++b) {
                const Iv br = block_sum(lead ? per[b].lead : per[b].trail);
                if (ge(add(cum, br), left)) break;
                cum = add(cum, br);
                st[2 * b + (lead ? 0 : 1)] = kFull;
            }
            if (b == nb) return;
            st[2 * b + (lead ? 0 : 1)] = cross(b, p, lead ? 0 : 1, cum, left);
        };
        const Iv first = lead_first ? tot.lead : tot.trail;
        if (ge(first, need)) {
            scan(lead_first, need);
            return;
        }
        for (u64 b = 0; b < nb; ++b) st[2 * b + (lead_first ? 0 : 1)] = kFull;
        scan(!lead_first, sub(need, first));
    }

    PlanResult run(u64* dec) {
        PlanResult pr;
        pr.block = block;
        pr.stops.assign(2 * nb, 0);
        auto finish = [&](int lp) {
            pr.last_plane = lp;
            if (o.on_last_plane && !o.fixed_plane) o.on_last_plane(lp);
            if (n > 0) {
                HostTrace ht("plan: decode_model");
                DevBuf<u64> ds(2 * nb, s);
                ds.upload(pr.stops.data(), 2 * nb);
                decode_model(m, n, block, lp, ds.p, dec, s);
                stream_sync(s);
            }
            return pr;
        };
        if (n == 0) return finish(63);
        if (o.fixed_plane) {  // factor streams: planes 63..fixed in full (core_codec.cpp:328-391)
            const int fp = *o.fixed_plane;
            pr.nplanes = 64 - fp;
            for (auto& v : pr.stops) v = kFull;
            return finish(fp);
        }
        HostTrace ht0("plan: initial sum");
        auto exact_sum = [&](int which) {  // which: -1 initial, else the recalibration at that plane
            if (ex_sums.empty()) {
                HostTrace ht("plan: exact sums (initial + recalibrations)");
                std::vector<std::pair<SumKind, int>> list{{SumKind::sq_backward, 0}};
                for (int q = 0; q < 64; ++q) list.push_back({SumKind::recal_backward, q});
                ex_sums = device_sums_serial(list, m, n, s);
            }
            return ex_sums[which < 0 ? 0 : 1 + which];
        };
        Iv tracked = exact ? pt(exact_sum(-1))
                           : from_sum(device_sum(SumKind::sq_backward, m, nullptr, n, 0, s), false);
        Iv ref = tracked;
        u64 terms = 0;
        const Iv tgt = pt(target);
        if (le(tracked, tgt)) return finish(63);  // nothing worth encoding
        Tot prev;
        bool have_prev = false;
        for (int p = 63; p >= 0; --p) {
            const PlaneBlockRec* per = stats(p, 0);
            Tot tot;
            for (u64 b = 0; b < nb; ++b) {
                tot.lead = add(tot.lead, block_sum(per[b].lead));
                tot.trail = add(tot.trail, block_sum(per[b].trail));
                tot.nlead += per[b].nlead;
                tot.nones += per[b].nones;
                tot.ntrail += per[b].ntrail;
            }
            const Iv red = add(tot.lead, tot.trail);
            ++pr.nplanes;
            if (le(sub(tracked, red), tgt)) {
                if (o.on_last_plane) o.on_last_plane(p);
                u64 ebits = 0;
                if (o.split && have_prev) {
                    HostTrace ht("plan: split probe emit");
                    if (o.probe) {
                        for (u64 e : probe_entropy_bytes(*o.probe, p + 1)) ebits += e * 8;
                    } else {
                        const auto er = emit_planes(m, nullptr, n, block, p + 1, p + 1, nullptr, o.coder, false, s);
                        for (u64 e : er.entropy_bytes) ebits += e * 8;
                    }
                }
                // the stats batch may have been replaced by the probe: refetch
                per = stats(p, 0);
                place_stops(p, sub(tracked, tgt), tot, per, have_prev ? &prev : nullptr, ebits, pr.stops);
                return finish(p);
            }
            tracked = sub(tracked, red);
            terms += tot.nones + tot.ntrail;
            const double c = 4.0 * std::numeric_limits<double>::epsilon() * static_cast<double>(terms);
            bool due;
            if (c * ref.lo > 0.1 * tracked.hi) due = true;
            else if (c * ref.hi <= 0.1 * tracked.lo) due = false;
            else {
                HostTrace ht("plan: ambiguous recalibration");
                throw Ambiguous{};
            }
            if (due) {
                HostTrace ht("plan: recalibration sum");
                tracked = exact ? pt(exact_sum(p))
                                : from_sum(device_sum(SumKind::recal_backward, m, nullptr, n, p, s), false);
                ref = tracked;
                terms = 0;
            }
            prev = tot;
            have_prev = true;
        }
        for (auto& v : pr.stops) v = kFull;
        return finish(0);
    }
};

void put_le(std::vector<u8>& o, u64 v, int bytes) {
    for (int i = 0; i < bytes; ++i) o.push_back(static_cast<u8>(v >> (8 * i)));
}

}  // namespace

u64 default_block(u64 n) { return std::max<u64>(4096, (n + 63) / 64); }

PlanResult plan_stream(const u64* m, u64 n, double target_int, const EncodeOpts& o, u64* dec, cudaStream_t s) {
    const u64 block = o.block ? o.block : default_block(n);
    const u64 nb = n == 0 ? 0 : (n + block - 1) / block;
    Planner pl{m, n, block, nb, target_int, o, false, s, {}, -1, 64};
    try {
        return pl.run(dec);
    } catch (const Ambiguous&) {
        Planner ex{m, n, block, nb, target_int, o, true, s, {}, -1, 64};
        PlanResult r = ex.run(dec);
        r.certified = false;
        r.fallbacks = 1;
        return r;
    }
}

std::vector<u8> finalize_stream(const u64* m, const u8* neg, u64 n, const PlanResult& pl, int coder, u64 count,
                                cudaStream_t s) {
    const u64 nb = n == 0 ? 0 : (n + pl.block - 1) / pl.block;
    std::vector<u8> o;
    put_le(o, count, 8);
    put_le(o, pl.block, 8);
    o.push_back(static_cast<u8>(pl.last_plane));
    put_le(o, nb, 4);
    for (u64 b = 0; b < nb; ++b) {
        put_le(o, pl.stops[2 * b], 8);
        put_le(o, pl.stops[2 * b + 1], 8);
    }
    put_le(o, static_cast<u64>(pl.nplanes), 4);
    if (pl.nplanes > 0 && nb > 0) {
        HostTrace ht("finalize: emit_planes");
        const auto er = emit_planes(m, neg, n, pl.block, pl.last_plane, 63, pl.stops.data(), coder, true, s);
        o.insert(o.end(), er.body.begin(), er.body.end());
    }
    return o;
}

}  // namespace tcb
