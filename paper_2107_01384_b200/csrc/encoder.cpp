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
#include <cstring>
#include <future>
#include <limits>

#include "encoder.hpp"
#include "exact.cuh"
#include "pipeline.hpp"

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
    // the first plane batch, launched before the initial backward sum (which
    // then runs on a side stream, its one-warp walk beside the batch's passes)
    std::unique_ptr<PlaneStatsJob> pre;
    int pre_p = -1;
    // The split probe's coder size bounds of the plane above the breakpoint the
    // sampled residuals predict, computed on a side stream while the exact plane
    // statistics run (used only when the exact breakpoint is the predicted one:
    // a full plane's sizes depend on nothing else).
    struct SpecProbe {
        int plane = -1;
        std::future<std::vector<u64>> fut;
        ~SpecProbe() {
            if (fut.valid()) fut.wait();
        }
    } spec;

    void speculate_probe(int plane) {
        if (spec.fut.valid() || plane > 63 || plane < 0 || !o.split || o.coder != 0 || o.probe ||
            (o.shard && o.shard->world > 1))
            return;
        // the highest priority (one above the call's stream): the probe's CTAs are
        // dispatched ahead of the plane statistics' as soon as they are enqueued
        static PerDevice<cudaStream_t> side_streams;
        cudaStream_t side = side_streams.get([] {
            int lo = 0, hi = 0;
            TCB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            cudaStream_t x;
            TCB_CUDA(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, hi));
            return x;
        });
        int dev = 0;
        TCB_CUDA(cudaGetDevice(&dev));
        EventHandle q;
        TCB_CUDA(cudaEventRecord(q.e, s));
        TCB_CUDA(cudaStreamWaitEvent(side, q.e, 0));
        spec.plane = plane;
        const u64* mm = m;
        const u64 nn = n, bl = block;
        // the caller waits until the probe's kernels are enqueued: queued ahead of
        // the plane statistics (same stream priority), its few CTAs start first and
        // the statistics fill the remaining SMs, instead of the probe waiting for
        // every statistics CTA to be dispatched
        auto enq = std::make_shared<std::promise<void>>();
        auto enq_f = enq->get_future();
        spec.fut = std::async(std::launch::async, [mm, nn, bl, plane, side, dev, enq] {
            bool sent = false;
            try {
                TCB_CUDA(cudaSetDevice(dev));
                auto r = entropy_size_bounds(mm, nn, bl, plane, side, {}, [&] {
                    sent = true;
                    enq->set_value();
                });
                if (!sent) enq->set_value();
                return r;
            } catch (...) {
                if (!sent) enq->set_value();
                throw;
            }
        });
        // TCB_PROBE_NOWAIT=1: rely on the side stream's priority alone (measurement switch:
        // c5 223.6 ms either way, the wait is off the critical path)
        static const bool nowait = std::getenv("TCB_PROBE_NOWAIT") != nullptr;
        if (!nowait) enq_f.wait();
    }

    // Exact statistics from plane p down: a sampled estimate of the residual
    // after each of the next 32 planes marks the likely breakpoint, and only the
    // planes down to it are computed exactly; a later plane triggers another batch.
    const PlaneStats& stats(int p) {
        if (!have[p]) {
            const int np = std::min(32, p + 1);
            HostTrace ht("plan: exact plane stats");
            const bool shd = o.shard && o.shard->world > 1;
            const BlockRange br = shd ? rank_blocks(nb, o.shard->world, o.shard->rank) : BlockRange{0, nb};
            std::unique_ptr<PlaneStatsJob> own;
            if (!(pre && pre_p == p)) own = std::make_unique<PlaneStatsJob>(m, n, block, p, np, s, br.b0, br.b1);
            PlaneStatsJob& job = own ? *own : *pre;
            int need = np;
            if (n > (u64{1} << 20)) {
                // the planes down to the first whose (sampled) residual is safely
                // below the target: the breakpoint is at or above it; a later plane
                // triggers another batch, so the estimate only affects the work
                auto res = job.approx_residuals();
                if (shd) {  // every rank sums the same partial estimates: the same `need` everywhere
                    DevBuf<double> dt(res.size(), s);
                    dt.upload(res.data(), res.size());
                    o.shard->allreduce_sum_f64(dt.p, res.size(), s);
                    res = dt.to_host();
                }
                for (int l = 0; l < np; ++l)
                    if (res[l] <= target / 1.02) {
                        need = std::min(np, l + 1);
                        if (l > 0) speculate_probe(p - l + 1);  // the probe plane of a breakpoint at p - l
                        break;
                    }
            }
            std::vector<ExOut> out = job.exact(need);
            if (!own) pre.reset();
            if (shd) {  // all-gather the ranks' blocks: out[k * nb + b] over every block
                const u64 nk = static_cast<u64>(2 * need);
                const std::vector<u8> mine(reinterpret_cast<const u8*>(out.data()),
                                           reinterpret_cast<const u8*>(out.data() + out.size()));
                const auto all = o.shard->allgather_blobs(mine, s);
                std::vector<ExOut> full(nk * nb);
                for (int r = 0; r < o.shard->world; ++r) {
                    const BlockRange rb = rank_blocks(nb, o.shard->world, r);
                    const u64 rn = rb.b1 - rb.b0;
                    if (all[r].size() != nk * rn * sizeof(ExOut)) throw Error("sharded compress: stats exchange");
                    const ExOut* src = reinterpret_cast<const ExOut*>(all[r].data());
                    for (u64 k = 0; k < nk; ++k)
                        for (u64 b = 0; b < rn; ++b) full[k * nb + rb.b0 + b] = src[k * rn + b];
                }
                out = std::move(full);
            }
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
    // the per-coefficient scan of block b from `cum` until cum >= need (by the
    // block's owner when sharded, then shared)
    ExOut cross(u64 b, int p, int term, double cum, double need) {
        HostTrace ht("plan: exact crossing scan");
        const bool shd = o.shard && o.shard->world > 1;
        const BlockRange br = shd ? rank_blocks(nb, o.shard->world, o.shard->rank) : BlockRange{0, nb};
        ExOut x{};
        const bool mine = b >= br.b0 && b < br.b1;
        if (mine)
            x = serial_sums(m, nullptr, {ExSeg{b * block, std::min(n, (b + 1) * block), 0, cum, need}}, {{term, p}},
                            s)[0];
        if (!shd) return x;
        std::vector<u8> blob;
        if (mine) blob.assign(reinterpret_cast<const u8*>(&x), reinterpret_cast<const u8*>(&x) + sizeof(x));
        for (const auto& bl : o.shard->allgather_blobs(blob, s))
            if (bl.size() == sizeof(ExOut)) std::memcpy(&x, bl.data(), sizeof(x));
        return x;
    }

    // the split-plane priority (core_codec.cpp:257-266) for a given entropy size of the previous plane
    static bool lead_first_for(const Tot& prev, u64 prev_ebits) {
        const double lead_cost = static_cast<double>(prev_ebits + prev.nones);
        const double trail_cost = static_cast<double>(prev.ntrail);
        const double eff_lead = lead_cost > 0 ? prev.lead / lead_cost : (prev.lead > 0 ? HUGE_VAL : 0.0);
        const double eff_trail = trail_cost > 0 ? prev.trail / trail_cost : (prev.trail > 0 ? HUGE_VAL : 0.0);
        return eff_lead >= eff_trail;
    }

    void place_stops(int p, double need, const Tot& tot, const PlaneStats& per, bool lead_first,
                     std::vector<u64>& stp) {
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
        double tracked;
        // off by default (TCB_SUM_OVERLAP=1): both are GPU-throughput-bound passes, so
        // running them side by side measured no faster than in sequence on c5
        static const bool overlap = std::getenv("TCB_SUM_OVERLAP") != nullptr;
        if (n > (u64{1} << 20) && overlap) {
            const bool shd = o.shard && o.shard->world > 1;
            const BlockRange br = shd ? rank_blocks(nb, o.shard->world, o.shard->rank) : BlockRange{0, nb};
            pre = std::make_unique<PlaneStatsJob>(m, n, block, 63, 32, s, br.b0, br.b1);
            pre_p = 63;
            static PerDevice<cudaStream_t> side_streams;
            cudaStream_t side = side_streams.get([] {
                cudaStream_t x;
                TCB_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
                return x;
            });
            EventHandle q;
            TCB_CUDA(cudaEventRecord(q.e, s));
            TCB_CUDA(cudaStreamWaitEvent(side, q.e, 0));
            HostTrace ht("plan: exact initial sum");
            tracked = serial_sums(m, nullptr, {ExSeg{0, n, 1, 0.0, HUGE_VAL}}, {{kExSq, 0}}, side)[0].sum;
        } else {
            tracked = full_sum(kExSq, 0);  // backward_sum_sse (core_codec.cpp:183)
        }
        double ref = tracked;
        u64 terms = 0;
        if (tracked <= target) return finish(63);  // nothing worth encoding
        Tot prev;
        bool have_prev = false;
        for (int p = 63; p >= 0; --p) {
            const PlaneStats& per = stats(p);
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
                if (o.on_breakpoint) o.on_breakpoint(p);
                bool lead_first = true;
                if (o.split && have_prev) {
                    HostTrace ht("plan: split probe emit");
                    const bool shd = o.shard && o.shard->world > 1;
                    const BlockRange br = shd ? rank_blocks(nb, o.shard->world, o.shard->rank) : BlockRange{0, nb};
                    // the ranks' sums of (lo, hi) or of exact sizes
                    auto all_sum = [&](std::vector<u64> v) {
                        if (!shd) return v;
                        const std::vector<u8> blob(reinterpret_cast<const u8*>(v.data()),
                                                   reinterpret_cast<const u8*>(v.data() + v.size()));
                        std::vector<u64> tot(v.size(), 0);
                        for (const auto& bl : o.shard->allgather_blobs(blob, s))
                            for (std::size_t i = 0; i < tot.size() && (i + 1) * sizeof(u64) <= bl.size(); ++i) {
                                u64 x;
                                std::memcpy(&x, bl.data() + i * sizeof(u64), sizeof(u64));
                                tot[i] += x;
                            }
                        return tot;
                    };
                    bool decided = false;
                    if (o.probe) {
                        u64 ebits = 0;
                        for (u64 e : probe_entropy_bytes(*o.probe, p + 1)) ebits += e * 8;
                        lead_first = lead_first_for(prev, ebits);
                        decided = true;
                    } else if (o.coder == 0) {
                        // the coder's size bounds from the model alone usually decide it
                        const auto b = spec.fut.valid() && spec.plane == p + 1
                                           ? spec.fut.get()
                                           : entropy_size_bounds(m, n, block, p + 1, s, br);
                        std::vector<u64> lh{0, 0};
                        for (std::size_t i = 0; i + 1 < b.size(); i += 2) {
                            lh[0] += b[i] * 8;
                            lh[1] += b[i + 1] * 8;
                        }
                        lh = all_sum(lh);
                        const bool a = lead_first_for(prev, lh[0]), z = lead_first_for(prev, lh[1]);
                        if (a == z) {
                            lead_first = a;
                            decided = true;
                        }
                    }
                    if (!decided) {  // the exact sizes: the full coder over plane p + 1
                        const auto er = emit_planes(m, nullptr, n, block, p + 1, p + 1, nullptr, o.coder, false, s, br);
                        u64 mine = 0;
                        for (u64 e : er.entropy_bytes) mine += e * 8;
                        lead_first = lead_first_for(prev, all_sum({mine})[0]);
                    }
                }
                place_stops(p, tracked - target, tot, per, lead_first, pr.stops);
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

namespace {
// (u32 size || payload) segments moved from the gathered per-rank bodies into
// container order (planes major, blocks minor), one CTA per segment
__global__ void gather_segments_kernel(const u8* __restrict__ src, u8* __restrict__ dst,
                                       const u64* __restrict__ tab /* src_off, dst_off, len */) {
    const u64 so = tab[3 * blockIdx.x], dof = tab[3 * blockIdx.x + 1], len = tab[3 * blockIdx.x + 2];
    for (u64 i = threadIdx.x; i < len; i += blockDim.x) dst[dof + i] = src[so + i];
}
}  // namespace

StreamParts finalize_stream_parts(const u64* m, const u8* neg, u64 n, const PlanResult& pl, int coder, u64 count,
                                  cudaStream_t s, const ShardComm* shard,
                                  const std::function<EmitDev*()>& upper) {
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
    if (pl.nplanes <= 0 || nb == 0) return out;
    HostTrace ht("finalize: emit_planes");
    if ((!shard || shard->world <= 1) && upper && pl.last_plane < 63) {
        // the full planes were coded beside the plan: code the last plane, append it
        EmitDev lo = emit_planes_device(m, neg, n, pl.block, pl.last_plane, pl.last_plane, pl.stops.data(), coder, s);
        EmitDev own;
        EmitDev* up = upper();
        if (!up) {
            own = emit_planes_device(m, neg, n, pl.block, pl.last_plane + 1, 63, nullptr, coder, s);
            up = &own;
        }
        out.body_size = up->size + lo.size;
        out.body = DevBuf<u8>(out.body_size + 1, s);
        if (up->size) TCB_CUDA(cudaMemcpyAsync(out.body.p, up->body.p, up->size, cudaMemcpyDeviceToDevice, s));
        if (lo.size)
            TCB_CUDA(cudaMemcpyAsync(out.body.p + up->size, lo.body.p, lo.size, cudaMemcpyDeviceToDevice, s));
        up->body.s = s;  // freed after the copy, in stream order
        return out;
    }
    if ((!shard || shard->world <= 1) && pl.nplanes >= 4 && n > (u64{1} << 20)) {
        // The range coder's time is set by the longest streams, which sit in the
        // densest planes: those planes are emitted, modelled and coded on this
        // (higher-priority) stream while the planes above and below them go
        // through the same steps on two side streams, instead of the longest
        // recurrences starting only after every plane's emission and model.
        const int lp = pl.last_plane;
        const auto hist = msb_histogram(m, n, pl.block, s);
        int best = lp;
        u64 bestc = 0;
        for (int p = lp; p <= 63; ++p) {
            u64 c = 0;
            for (u64 b = 0; b < nb; ++b) c = std::max(c, hist[b * 65 + static_cast<u64>(p + 1)]);
            if (c > bestc) {
                bestc = c;
                best = p;
            }
        }
        const int h_lo = std::max(lp, best - 1), h_hi = std::min(63, best + 1);
        // the planes above and below the densest ones, each on its own side stream
        // (driven by its own thread), all three groups started together
        // (the planes below are dense too: their stream at the call's priority; the
        // sparse planes above at the lowest)
        static PerDevice<std::pair<cudaStream_t, cudaStream_t>> side_streams;
        const auto sides = side_streams.get([] {
            int lo = 0, hi = 0;
            TCB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            std::pair<cudaStream_t, cudaStream_t> x;
            TCB_CUDA(cudaStreamCreateWithPriority(&x.first, cudaStreamNonBlocking, lo));
            TCB_CUDA(cudaStreamCreateWithPriority(&x.second, cudaStreamNonBlocking, hi < lo ? hi + 1 : hi));
            return x;
        });
        const int dev = cur_device();
        EventHandle q;
        TCB_CUDA(cudaEventRecord(q.e, s));
        TCB_CUDA(cudaStreamWaitEvent(sides.first, q.e, 0));
        TCB_CUDA(cudaStreamWaitEvent(sides.second, q.e, 0));
        auto run = [&, dev](int lo_p, int hi_p, const u64* stops, cudaStream_t st) {
            return std::async(std::launch::async, [&, dev, lo_p, hi_p, stops, st] {
                TCB_CUDA(cudaSetDevice(dev));
                EmitDev e;
                if (lo_p <= hi_p) e = emit_planes_device(m, neg, n, pl.block, lo_p, hi_p, stops, coder, st, {}, &hist);
                return e;
            });
        };
        auto f_up = run(h_hi + 1, 63, nullptr, sides.first);
        auto f_lo = run(lp, h_lo - 1, pl.stops.data(), sides.second);
        EmitDev mid = emit_planes_device(m, neg, n, pl.block, h_lo, h_hi, h_lo == lp ? pl.stops.data() : nullptr,
                                         coder, s, {}, &hist);
        EmitDev up = f_up.get(), lo = f_lo.get();
        for (cudaStream_t st : {sides.first, sides.second}) {  // their assembly kernels, before the copies
            EventHandle fin;
            TCB_CUDA(cudaEventRecord(fin.e, st));
            TCB_CUDA(cudaStreamWaitEvent(s, fin.e, 0));
        }
        out.body_size = up.size + mid.size + lo.size;
        out.body = DevBuf<u8>(out.body_size + 1, s);
        u64 at = 0;
        for (EmitDev* e : {&up, &mid, &lo}) {  // container order: planes from the top down
            if (e->size) TCB_CUDA(cudaMemcpyAsync(out.body.p + at, e->body.p, e->size, cudaMemcpyDeviceToDevice, s));
            at += e->size;
            e->body.s = s;  // freed after the copy, in stream order
        }
        return out;
    }
    if (!shard || shard->world <= 1) {
        EmitDev er = emit_planes_device(m, neg, n, pl.block, pl.last_plane, 63, pl.stops.data(), coder, s);
        out.body = std::move(er.body);
        out.body_size = er.size;
        return out;
    }
    // sharded: every rank emits and codes its own blocks of every plane; the
    // segments are gathered and put in container order (the result is complete
    // on every rank; rank 0 writes the container)
    const int P = shard->world;
    const BlockRange br = rank_blocks(nb, P, shard->rank);
    EmitDev er = emit_planes_device(m, neg, n, pl.block, pl.last_plane, 63, pl.stops.data(), coder, s, br);
    const std::vector<u8> mine(reinterpret_cast<const u8*>(er.stream_bytes.data()),
                               reinterpret_cast<const u8*>(er.stream_bytes.data() + er.stream_bytes.size()));
    const auto sizes = shard->allgather_blobs(mine, s);
    u64 mx = 0;
    std::vector<u64> rank_total(P, 0);
    for (int r = 0; r < P; ++r) {
        const u64* z = reinterpret_cast<const u64*>(sizes[r].data());
        for (u64 i = 0; i < sizes[r].size() / sizeof(u64); ++i) rank_total[r] += z[i];
        mx = std::max(mx, rank_total[r]);
    }
    DevBuf<u8> send(mx + 1, s), recv((mx + 1) * P, s);
    if (er.size) TCB_CUDA(cudaMemcpyAsync(send.p, er.body.p, er.size, cudaMemcpyDeviceToDevice, s));
    shard->allgather(send.p, recv.p, mx + 1, s);
    // copy table: stream (plane pi, block b) of rank r sits at local index pi * nb_r + (b - b0_r)
    const u64 np = static_cast<u64>(pl.nplanes);
    std::vector<std::vector<u64>> loc_off(P);
    for (int r = 0; r < P; ++r) {
        const u64* z = reinterpret_cast<const u64*>(sizes[r].data());
        const u64 cnt = sizes[r].size() / sizeof(u64);
        loc_off[r].resize(cnt);
        u64 acc = 0;
        for (u64 i = 0; i < cnt; ++i) {
            loc_off[r][i] = acc;
            acc += z[i];
        }
    }
    std::vector<u64> tab;
    tab.reserve(3 * np * nb);
    u64 dst = 0;
    for (u64 pi = 0; pi < np; ++pi)
        for (u64 b = 0; b < nb; ++b) {
            int r = 0;
            while (r + 1 < P && rank_blocks(nb, P, r + 1).b0 <= b) ++r;
            const BlockRange rb = rank_blocks(nb, P, r);
            const u64 i = pi * (rb.b1 - rb.b0) + (b - rb.b0);
            const u64 len = reinterpret_cast<const u64*>(sizes[r].data())[i];
            tab.push_back(static_cast<u64>(r) * (mx + 1) + loc_off[r][i]);
            tab.push_back(dst);
            tab.push_back(len);
            dst += len;
        }
    DevBuf<u64> dtab(tab.size(), s);
    dtab.upload(tab.data(), tab.size());
    out.body = DevBuf<u8>(dst + 1, s);
    out.body_size = dst;
    gather_segments_kernel<<<static_cast<unsigned>(np * nb), 256, 0, s>>>(recv.p, out.body.p, dtab.p);
    count_launch();
    TCB_LAUNCH();
    stream_sync(s);
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
