// Breakpoint logic of the device encoder (corecodec::Encoder::plan and
// place_stops, core_codec.cpp:173-342, with error_model.cpp:34-72).
//
// The reference decides the breakpoint plane, the recalibration points and the
// split-plane stops by comparing doubles it accumulates SERIALLY.  Every such
// double is obtained here bit for bit from the exact serial-sum engine
// (exact.cu: binade-local unit arithmetic with a parity transducer, composed
// in parallel), so the host replays the reference's decisions on the very
// same doubles: no tolerance, no certification, no fallback.
// TCB_EXACT_REFERENCE=1 computes the same sums with the plain one-thread
// serial chain instead (verification).
//
// This TU must not be compiled with FMA contraction (host x86-64: no -mfma).
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <limits>

#include "encoder.hpp"
#include "exact.cuh"

namespace tcb {

namespace {

std::vector<ExOut> serial_sums(const u64* m, const u64* dec, const std::vector<ExSeg>& segs,
                               const std::vector<ExKind>& kinds, cudaStream_t s) {
    return exact_serial(m, dec, segs, kinds, s);
}

struct PlaneStats {  // build_block statistics of one plane, per block (core_codec.cpp:131-155)
    std::vector<double> lead, trail;
    std::vector<u64> nlead, nones, ntrail;
};

struct Tot {  // PlaneBlockStats totals, summed over blocks in block order (core_codec.cpp:210-218)
    double lead = 0.0, trail = 0.0;
    u64 nlead = 0, nones = 0, ntrail = 0;
};

struct Planner {
    const u64* m;
    u64 n, block, nb;
    double target;
    EncodeOpts o;
    cudaStream_t s;
    std::vector<PlaneStats> st = std::vector<PlaneStats>(64);
    std::vector<char> have = std::vector<char>(64, 0);

    // Exact statistics from plane p down: 32 planes' approximate totals first,
    // the approximate `tracked` trajectory from the current (exact) value marks
    // the likely breakpoint, and only the planes down to it (+2) are computed
    // exactly; a later plane triggers another batch.
    const PlaneStats& stats(int p, double tracked_now) {
        if (!have[p]) {
            const int np = std::min(32, p + 1);
            HostTrace ht("plan: exact plane stats");
            PlaneStatsJob job(m, n, block, p, np, s);
            int need = np;
            if (n > (u64{1} << 20)) {
                const auto tot = job.approx_totals();
                double tr = tracked_now;
                for (int l = 0; l < np; ++l) {
                    const double red = tot[2 * l] + tot[2 * l + 1];
                    if (tr - red <= target * (1.0 + 1e-6)) {
                        need = std::min(np, l + 3);
                        break;
                    }
                    tr -= red;
                }
            }
            const auto out = job.exact(need);
            for (int l = 0; l < need; ++l) {
                const int q = p - l;
                const u64 kl = static_cast<u64>(2 * l), kt = kl + 1;
                PlaneStats& ps = st[q];
                ps.lead.resize(nb);
                ps.trail.resize(nb);
                ps.nlead.resize(nb);
                ps.nones.resize(nb);
                ps.ntrail.resize(nb);
                for (u64 b = 0; b < nb; ++b) {
                    const ExOut& L = out[kl * nb + b];
                    const ExOut& T = out[kt * nb + b];
                    ps.lead[b] = L.sum;
                    ps.trail[b] = T.sum;
                    ps.nlead[b] = L.c0;
                    ps.nones[b] = L.c1;
                    ps.ntrail[b] = T.c1;
                }
                have[q] = 1;
            }
        }
        return st[p];
    }
    double full_sum(int term, int plane) {  // a backward sum over the whole core
        HostTrace ht(term == kExSq ? "plan: exact initial sum" : "plan: exact recalibration sum");
        return serial_sums(m, nullptr, {ExSeg{0, n, 1, 0.0, HUGE_VAL}}, {{term, plane}}, s)[0].sum;
    }
    // the per-coefficient scan of block b from `cum` until cum >= need
    ExOut cross(u64 b, int p, int term, double cum, double need) {
        HostTrace ht("plan: exact crossing scan");
        return serial_sums(m, nullptr, {ExSeg{b * block, std::min(n, (b + 1) * block), 0, cum, need}}, {{term, p}},
                           s)[0];
    }

    void place_stops(int p, double need, const Tot& tot, const PlaneStats& per, const Tot* prev, u64 prev_ebits,
                     std::vector<u64>& stp) {
        bool lead_first = true;
        if (o.split && prev) {
            const double lead_cost = static_cast<double>(prev_ebits + prev->nones);
            const double trail_cost = static_cast<double>(prev->ntrail);
            const double eff_lead = lead_cost > 0 ? prev->lead / lead_cost : (prev->lead > 0 ? HUGE_VAL : 0.0);
            const double eff_trail = trail_cost > 0 ? prev->trail / trail_cost : (prev->trail > 0 ? HUGE_VAL : 0.0);
            lead_first = eff_lead >= eff_trail;
        }
        if (!o.split) {
            double cum = 0;
            u64 b = 0;
            for (; b < nb; ++b) {
                const double br = per.lead[b] + per.trail[b];
                if (cum + br >= need) break;
                cum += br;
                stp[2 * b] = stp[2 * b + 1] = kFull;
            }
            if (b == nb) return;
            const ExOut x = cross(b, p, kExBoth, cum, need);
            stp[2 * b] = x.c0;
            stp[2 * b + 1] = x.c1;
            return;
        }
        auto scan = [&](bool lead, double left) {
            double cum = 0;
            u64 b = 0;
            for (; b < nb; ++b) {
                const double br = lead ? per.lead[b] : per.trail[b];
                if (cum + br >= left) break;
                cum += br;
                stp[2 * b + (lead ? 0 : 1)] = kFull;
            }
            if (b == nb) return;
            const ExOut x = cross(b, p, lead ? kExLead : kExTrail, cum, left);
            stp[2 * b + (lead ? 0 : 1)] = lead ? x.c0 : x.c1;
        };
        const double first = lead_first ? tot.lead : tot.trail;
        if (first >= need) {
            scan(lead_first, need);
            return;
        }
        for (u64 b = 0; b < nb; ++b) stp[2 * b + (lead_first ? 0 : 1)] = kFull;
        scan(!lead_first, need - first);
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
        double tracked = full_sum(kExSq, 0);  // backward_sum_sse (core_codec.cpp:183)
        double ref = tracked;
        u64 terms = 0;
        if (tracked <= target) return finish(63);  // nothing worth encoding
        Tot prev;
        bool have_prev = false;
        for (int p = 63; p >= 0; --p) {
            const PlaneStats& per = stats(p, tracked);
            Tot tot;
            for (u64 b = 0; b < nb; ++b) {
                tot.lead += per.lead[b];
                tot.trail += per.trail[b];
                tot.nlead += per.nlead[b];
                tot.nones += per.nones[b];
                tot.ntrail += per.ntrail[b];
            }
            const double red = tot.lead + tot.trail;
            ++pr.nplanes;
            if (tracked - red <= target) {
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
                place_stops(p, tracked - target, tot, per, have_prev ? &prev : nullptr, ebits, pr.stops);
                return finish(p);
            }
            tracked -= red;
            terms += tot.nones + tot.ntrail;
            // recalibration_due (error_model.cpp:43-52)
            const double margin = 4.0 * std::numeric_limits<double>::epsilon() * static_cast<double>(terms) * ref;
            if (margin > 0.1 * tracked) {
                tracked = full_sum(kExRecal, p);
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
    Planner pl{m, n, block, nb, target_int, o, s};
    return pl.run(dec);
}

StreamParts finalize_stream_parts(const u64* m, const u8* neg, u64 n, const PlanResult& pl, int coder, u64 count,
                                  cudaStream_t s) {
    const u64 nb = n == 0 ? 0 : (n + pl.block - 1) / pl.block;
    StreamParts out;
    std::vector<u8>& o = out.head;
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
        EmitDev er = emit_planes_device(m, neg, n, pl.block, pl.last_plane, 63, pl.stops.data(), coder, s);
        out.body = std::move(er.body);
        out.body_size = er.size;
    }
    return out;
}

std::vector<u8> finalize_stream(const u64* m, const u8* neg, u64 n, const PlanResult& pl, int coder, u64 count,
                                cudaStream_t s) {
    StreamParts p = finalize_stream_parts(m, neg, n, pl, coder, count, s);
    std::vector<u8> o = std::move(p.head);
    const std::size_t h = o.size();
    o.resize(h + p.body_size);
    if (p.body_size) p.body.download(o.data() + h, p.body_size);
    stream_sync(s);
    return o;
}

}  // namespace tcb
