#!/usr/bin/env python
"""Compress-throughput benchmark (BASELINE.json metric) for the B200 path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Headline workload (BASELINE.json configs[4], the config the metric is quoted
on at 1/2/4/8 B200): c5 = 1024^3 fp32 Gaussian random field, E(k) ~ k^-5/3 for
k <= 341, seeded torch FFT on the GPU (synthetic: the paper's datasets are not
available), requested relative error 1e-2, reference-default parameters
(fp64 internal, rtmss 0.5, AC coder, split planes).  A step = one
pipeline::compress of that tensor (device-resident input -> container bytes in
host memory).  The input is 4 GiB (> the 126 MB L2), so no flush is needed.
The same JSON line carries c5 @ 1e-3 and c2 (256^3 fp64 @ 1e-4) as secondary
device-resident measurements.  N > 1: the ranks compress ONE c5 tensor sharded
along its last processed mode (strong scaling; NCCL all-reduce of partial
Grams), max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "c5: 1024^3 fp32 Gaussian random field E(k)~k^-5/3 (k<=341), seeded torch FFT, RE 1e-2"
C2_WORKLOAD = "c2: 256^3 fp64, 64 separable k^-1.5 sinusoid terms + N(0,1e-5), RE 1e-4"
CPU_SAMPLE_N = 384  # bounded CPU sample: the c5 generator at 384^3 (kmax = n/3)
METRIC = "compress throughput GB/s (input bytes)"
STAGES = ["ingest", "permute", "gram", "eig", "ttm", "quant", "stats", "emit", "ac", "factor", "sum", "tc"]


def _config(re):
    """The workload description, identical on both arms (the driver compares the dicts)."""
    return {"workload": WORKLOAD, "re": re, "l2": "input 4 GiB > L2 (no flush needed)"}


def round_up(a, b):
    return (a + b - 1) // b * b


def _env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def _ncu_traffic(kernel, nth=0):
    """DRAM bytes (read + write) of the nth launch of `kernel` in the committed
    ncu --set full summary of one c5 compress (profiles/), or None."""
    import glob

    for path in sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                              "ncu_*_full_summary.txt")), reverse=True):
        for line in open(path):
            f = line.split()
            if f and f[0] == kernel and len(f) > 5:
                if nth > 0:
                    nth -= 1
                    continue
                try:
                    return float(f[5]) * 1e6
                except ValueError:
                    break
    return None


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, in process via
    NVML (no nvidia-smi fork inside the timed region), nvidia-smi as a fallback."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = [getattr(pynvml, n, 0) for n in ("nvmlClocksEventReasonHwSlowdown",
                                                    "nvmlClocksEventReasonHwThermalSlowdown",
                                                    "nvmlClocksEventReasonSwThermalSlowdown",
                                                    "nvmlClocksEventReasonSwPowerCap")]
            bits = [b or d for b, d in zip(bits, (0x8, 0x40, 0x20, 0x4))]
            reasons_fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def sample():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = reasons_fn(h)
                return [str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits]
        except Exception:
            sample = None

        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    if sample is not None:
                        self.samples.append(sample())
                    else:
                        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                             timeout=5).stdout.strip()
                        if out:
                            self.samples.append([v.strip() for v in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.02 if sample is not None else 0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def algorithmic_work(shape, ranks, order):
    """Gram flops (SYRK lower-triangle count), TTM flops, per SURVEY.md 8(d)."""
    cur = [shape[p] for p in order]
    gram = ttm = 0.0
    for step, mode in enumerate(order):
        rows = cur[0]
        cols = int(np.prod(cur)) // rows
        r = ranks[mode]
        if rows <= cols:
            gram += rows * (rows + 1) * cols
        else:
            gram += cols * (cols + 1) * rows + 2.0 * rows * cols * r
        ttm += 2.0 * rows * cols * r
        cur = cur[1:] + [r]
    return gram, ttm


def cpu_reference_step(x, re):
    import oracle

    t0 = time.perf_counter()
    info = oracle.compress(x, target_re=re)
    return time.perf_counter() - t0, info


def c5_tensor(n=1024, seed=0):
    """c5 (or its n^3 sample): the BASELINE GRF generator on the GPU, float32, kmax = n // 3."""
    import synth

    return synth.grf_torch(n=n, kmax=n // 3, seed=seed)


def cpu_sample(seed=0):
    """The bounded CPU sample of the c5 workload: the same generator at 384^3 (1/19 of the bytes; the
    per-byte Gram/TTM work grows with the mode size, so this overstates the CPU's c5 throughput)."""
    return c5_tensor(CPU_SAMPLE_N, seed).cpu().numpy()


def run_reference(args):
    rank, _, world = _env_rank()
    if rank != 0:
        return
    import oracle

    nth = oracle.threads()
    x = cpu_sample()
    nbytes = x.nbytes
    for _ in range(args.warmup):
        cpu_reference_step(x, args.re)
    times = []
    for _ in range(args.steps):
        dt, info = cpu_reference_step(x, args.re)
        times.append(dt)
    tot = sum(times)
    value = nbytes * len(times) / tot / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(args.re),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": nth, "kind": "port",
                         "sample": f"each step one full compress of the c5 generator at {CPU_SAMPLE_N}^3 "
                                   f"({nbytes} B, RE {args.re}) by oracle/ (restatement of the reference path, "
                                   f"integer half pinned to the reference's own code; Gram and projection loops "
                                   f"OpenMP-parallel over {nth} host threads)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def c2_slab(world, rank, seed=0):
    """Rank `rank`'s 256^3 slab (along mode 2) of the weak-scaled c2-family
    tensor 256 x 256 x (256 world)."""
    rng = np.random.default_rng(seed)
    shape = (256, 256, 256 * world)
    K = 64
    amps = np.arange(1, K + 1, dtype=np.float64) ** -1.5
    mats = [np.empty((n, K)) for n in shape]
    for k in range(K):
        for m, n in enumerate(shape):
            f = rng.uniform(0.5, 4.0)
            ph = rng.uniform(0.0, 2 * np.pi)
            mats[m][:, k] = np.sin(2 * np.pi * f * (np.arange(n, dtype=np.float64) / n) + ph)
    v3 = mats[2][rank * 256:(rank + 1) * 256]
    rest = (mats[1][:, None, :] * v3[None, :, :]).reshape(-1, K)
    slab = ((mats[0] * amps[None, :]) @ rest.T).reshape(256, 256, 256)
    slab += 1e-5 * np.random.default_rng(seed * 7919 + 1 + rank).standard_normal(slab.shape)
    return np.ascontiguousarray(slab)


def main_sharded(args, rank, local, world):
    """N ranks compress ONE c5 tensor (1024^3 fp32) sharded along its last
    processed mode: rank k holds slab k of mode 2 (library path: partial Grams
    all-reduced over NCCL, replicated eigensolve, shard-local TTM, gather before
    the last step).  Strong scaling: value = 4 GiB / max-over-ranks time."""
    import torch
    import torch.distributed as dist

    import paper_2107_01384_b200 as tcb
    from paper_2107_01384_b200 import shard

    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    full = c5_tensor()
    shape = list(full.shape)
    lo, hi = shard.shard_bounds(shape[2], world, rank)
    xs = full[:, :, lo:hi].contiguous()
    del full
    torch.cuda.empty_cache()
    total_bytes = 4 * shape[0] * shape[1] * shape[2]
    params = tcb.Params(target_re=args.re)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step(x):
        return shard.compress_sharded(x, shape, tcb.Dtype.float32, params)

    for _ in range(args.warmup):
        res = step(xs)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = tcb.kernel_launches()
    step_ms = []
    for _ in range(args.steps):
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        res = step(xs)
        b.record()
        b.synchronize()
        step_ms.append(a.elapsed_time(b))
    barrier()
    launches = (tcb.kernel_launches() - launches0) // max(1, args.steps)
    host = xs.cpu().pin_memory()
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 5))):  # this rank's slab from pinned host memory
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        r2 = step(host.to(dev, non_blocking=True))
        b.record()
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    barrier()
    clk = clocks.stop()
    t = torch.tensor([sum(step_ms) / len(step_ms), sum(e2e_ms) / len(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, ms_e2e = float(t[0]), float(t[1])
    value = total_bytes / (ms * 1e-3) / 1e9
    e2e = total_bytes / (ms_e2e * 1e-3) / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(args.re),
            "result": {"input_bytes": total_bytes, "ranks": res.ranks, "container_bytes": len(res.container)},
            "parallelism": f"shard mode 2 over {world} ranks (NCCL all-reduce of partial Grams, "
                           f"replicated eigensolve, shard-local TTM and block-sharded encoding)",
            "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": int(host.numel() * 4),
                    "d2h_bytes_per_step": len(r2.container)},
            "gpu_launches": int(launches),
            "cpu_baseline": None,
            "clocks": clk,
            "step_ms_all": [round(v, 3) for v in step_ms],
            "e2e_ms_all": [round(v, 3) for v in e2e_ms],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def device_steps(tcb, x_dev, nbytes, dtype, shape, params, steps, warmup):
    """compress_device on a resident input: per-step CUDA events (the input exceeds L2)."""
    import torch

    res = None
    for _ in range(warmup):
        res = tcb.compress_device(x_dev.data_ptr(), nbytes, dtype, shape, params)
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        raw = tcb.compress_device_raw(x_dev.data_ptr(), nbytes, dtype, shape, params)
        b.record()  # the container is in host memory: the library returned it
        b.synchronize()
        ms.append(a.elapsed_time(b))
        res = tcb._result(raw)  # (copied into a Python bytes object outside the timed region)
    return res, ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--re", type=float, default=1e-2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="sharded one-tensor path also at N=1")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    rank, local, world = _env_rank()
    import torch

    torch.cuda.set_device(local)
    if world > 1 or args.sharded:
        main_sharded(args, rank, local, world)
        return

    import ctypes as C

    import paper_2107_01384_b200 as tcb
    import synth

    dev = torch.device("cuda", local)
    L = tcb.lib()
    x = c5_tensor()
    shape = list(x.shape)
    nbytes = x.numel() * 4
    params = tcb.Params(target_re=args.re)

    clocks = ClockSampler(local)
    clocks.start()
    launches0 = tcb.kernel_launches()
    res, step_ms = device_steps(tcb, x, nbytes, tcb.Dtype.float32, shape, params, args.steps, args.warmup)
    launches = (tcb.kernel_launches() - launches0) // max(1, args.steps + args.warmup)
    # ---- end to end through the public host API: pinned input bytes in, container bytes out
    host = x.cpu().pin_memory()
    src = tcb.SourceBuffer(memoryview(host.numpy()).cast("B"), tcb.Dtype.float32, shape)
    # W warm-up + K timed steps of one identical loop (events, synchronisation and
    # frees included), the first W discarded
    e2e_ms, e2e_bytes = [], []
    for it in range(args.warmup + args.steps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        raw = tcb.compress_raw(src, params)  # tcb_compress: returns with the container in host memory
        b.record()
        b.synchronize()
        if it >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
            e2e_bytes.append(int(raw.container_size))
        tcb.free_raw(raw)
    # the Python mirror's compress() on top: the container copied into a Python bytes
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    r2 = tcb.compress(src, params)
    b.record()
    b.synchronize()
    py_ms = a.elapsed_time(b)
    assert len(r2.container) == e2e_bytes[-1]
    clk = clocks.stop()
    del host, src
    tot = float(sum(step_ms))
    value = nbytes * args.steps / (tot * 1e-3) / 1e9
    e2e = nbytes * len(e2e_ms) / (sum(e2e_ms) * 1e-3) / 1e9

    # ---- per-stage breakdown (one extra step with stages run sequentially and timed)
    L.tcb_prof_enable(1)
    torch.cuda.synchronize()
    res_p = tcb.compress_device(x.data_ptr(), nbytes, tcb.Dtype.float32, shape, params)
    L.tcb_prof_enable(0)
    ms = (C.c_double * len(STAGES))()
    cnt = (C.c_uint64 * len(STAGES))()
    L.tcb_prof_read(ms, cnt, len(STAGES))
    stage_ms = {s: round(ms[i], 3) for i, s in enumerate(STAGES)}
    L.tcb_peak_dmma_tflops.restype = C.c_double
    dmma_peak = float(L.tcb_peak_dmma_tflops())
    peaks, peak_src = _peaks()
    order = [0, 1, 2]
    gram_flop, ttm_flop = algorithmic_work(shape, res.ranks, order)

    # ---- the dominant launches, timed live on the launching stream (tcb_prof events):
    # mode 0's Gram and TTM exactly as the pipeline runs them on c5 (fp64 unfolding ->
    # Ozaki digit slices -> tcgen05 kind::i8 products in TMEM -> exact int64 combine),
    # on the fp64 cast of the resident input; "tc" = the tcgen05 kernel alone
    x64 = x.double()
    rows0, cols0, r0 = shape[0], nbytes // 4 // shape[0], res.ranks[0]
    u0 = torch.linalg.qr(torch.randn(rows0, r0, dtype=torch.float64, device=dev))[0].contiguous()
    nxt = torch.empty(cols0 * r0, dtype=torch.float64, device=dev)
    g0 = torch.empty(rows0 * rows0, dtype=torch.float64, device=dev)
    L.tcb_dev_gram_ozaki.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
    L.tcb_dev_ttm_ozaki.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p]

    def timed(fn, stages, reps=3):
        out = {k: [] for k in stages}
        for _ in range(reps):
            torch.cuda.synchronize()
            L.tcb_prof_enable(1)
            assert fn() == 0
            L.tcb_prof_enable(0)
            L.tcb_prof_read(ms, cnt, len(STAGES))
            for k in stages:
                out[k].append(ms[STAGES.index(k)])
        return {k: float(np.median(v)) for k, v in out.items()}

    tt = timed(lambda: L.tcb_dev_ttm_ozaki(x64.data_ptr(), rows0, cols0, u0.data_ptr(), r0, nxt.data_ptr()),
               ["ttm", "tc"])
    tg = timed(lambda: L.tcb_dev_gram_ozaki(x64.data_ptr(), rows0, cols0, g0.data_ptr()), ["gram", "tc"])
    del x64, nxt, g0
    torch.cuda.empty_cache()
    ttm_flop0 = 2.0 * rows0 * cols0 * r0
    gram_flop0 = float(rows0 * (rows0 + 1) * cols0)
    pairs = 15  # digit-slice pairs (s, t) with s + t <= 4 (five slices)
    int8_peak = 2.0 * float(peaks.get("bf16_tflops", 1652.1))
    ttm_ops, gram_ops = pairs * ttm_flop0, pairs * gram_flop0
    ach = ttm_ops / (tt["tc"] * 1e-3) / 1e12
    roof = {"kernel": "oz_mma_kernel (tcgen05.mma kind::i8, TMA-staged, 5 int32 accumulators in TMEM) for the "
                      "mode-0 TTM, 1048576 x r0 by 1024 x 5 digit slices, median of 3 live launches",
            "bound": "tensor", "achieved": ach, "peak": int8_peak, "unit": "TOP/s (int8)", "frac": ach / int8_peak,
            # one c5 compress launches oz_mma_kernel as Gram 0, TTM 0, Gram 1, ...: the 2nd is this one
            "traffic": _ncu_traffic("oz_mma_kernel", 1),
            "traffic_algorithmic": float(5 * round_up(rows0, 128) * cols0 + 8 * cols0 * r0),
            "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of the mode-0 TTM launch, ncu --set full "
                              "(profiles/ncu_r02_full_summary.txt); algorithmic = the unfolding's five digit slices "
                              "read once + the fp64 output written once",
            "ops": ttm_ops, "ms": tt["tc"],
            "peak_source": "2 x measured bf16 burst (MEASURED_PEAKS.json): B200 int8 dense runs at twice bf16",
            "work": "15 slice-pair products of the TTM: 15 * 2 * rows * cols * r int8 ops (algorithmic)",
            "fp64_equivalent": {"flop": ttm_flop0, "ms_with_split_and_combine": tt["ttm"],
                                "tflops": ttm_flop0 / (tt["ttm"] * 1e-3) / 1e12, "dmma_peak": dmma_peak,
                                "frac_of_dmma_peak": ttm_flop0 / (tt["ttm"] * 1e-3) / 1e12 / dmma_peak},
            "gram_mode0": {"ops": gram_ops, "ms_tc": tg["tc"], "tops": gram_ops / (tg["tc"] * 1e-3) / 1e12,
                           "frac": gram_ops / (tg["tc"] * 1e-3) / 1e12 / int8_peak,
                           "work": "15 * rows * (rows + 1) * cols (SYRK count per slice pair)",
                           "ms_with_split_and_combine": tg["gram"],
                           "fp64_equivalent_tflops": gram_flop0 / (tg["gram"] * 1e-3) / 1e12,
                           "frac_of_dmma_peak": gram_flop0 / (tg["gram"] * 1e-3) / 1e12 / dmma_peak},
            "all_modes": {"gram_flop": gram_flop, "gram_ms": stage_ms["gram"], "ttm_flop": ttm_flop,
                          "ttm_ms": stage_ms["ttm"], "tc_ms": stage_ms.get("tc"),
                          "fp64_equivalent_frac_of_dmma_peak": (gram_flop + ttm_flop)
                          / max(stage_ms["gram"] + stage_ms["ttm"], 1e-9) / 1e9 / dmma_peak}}
    # encoder: B_enc = 2 * 8 * N_core + payload over the stats+emit+ac stages, against HBM
    n_core = int(np.prod(res.ranks))
    b_enc = 2 * 8 * n_core + len(res.container)
    enc_ms = stage_ms["stats"] + stage_ms["emit"] + stage_ms["ac"] + stage_ms["quant"]
    roof["encoder"] = {"bytes": b_enc, "ms": enc_ms, "gbs": b_enc / max(enc_ms, 1e-9) / 1e6,
                       "peak_gbs": peaks.get("hbm_gbs"), "frac": b_enc / max(enc_ms, 1e-9) / 1e6 /
                       float(peaks.get("hbm_gbs", 6553.6)), "peak_source": peak_src,
                       "note": "quantise + exact statistics + emission + range coding of the core "
                               "(sequential profiled step); the range coder is serial per stream"}
    roof["eig"] = {"ms": stage_ms["eig"], "note": "latency-bound (tridiagonalisation steps)"}

    # ---- secondary lines: c5 @ 1e-3 and c2 @ 1e-4, device-resident
    secondary = {}
    if not args.no_secondary:
        r3, ms3 = device_steps(tcb, x, nbytes, tcb.Dtype.float32, shape, tcb.Params(target_re=1e-3),
                               max(2, args.steps // 4), 1)
        secondary["c5_re1e-3"] = {"value": nbytes * len(ms3) / (sum(ms3) * 1e-3) / 1e9, "unit": "GB/s",
                                  "ms_per_step": sum(ms3) / len(ms3), "ranks": r3.ranks,
                                  "container_bytes": len(r3.container), "steps": len(ms3)}
    del x
    torch.cuda.empty_cache()
    if not args.no_secondary:
        xc2 = synth.make("c2", seed=0)
        d2 = torch.from_numpy(xc2.view(np.uint8).reshape(-1)).to(dev)
        rc2, msc2 = device_steps(tcb, d2, xc2.nbytes, tcb.Dtype.float64, list(xc2.shape),
                                 tcb.Params(target_re=1e-4), max(5, args.steps), 2)
        secondary["c2_re1e-4"] = {"workload": C2_WORKLOAD, "value": xc2.nbytes * len(msc2) / (sum(msc2) * 1e-3)
                                  / 1e9, "unit": "GB/s", "ms_per_step": sum(msc2) / len(msc2),
                                  "ranks": rc2.ranks, "container_bytes": len(rc2.container), "steps": len(msc2)}
        del d2

    # ---- CPU baseline (rank 0, N=1): the oracle on the bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        xs = cpu_sample()
        ts = []
        t_start = time.perf_counter()
        while time.perf_counter() - t_start < 10.0 or not ts:
            dt, _ = cpu_reference_step(xs, args.re)
            ts.append(dt)
        nth = oracle.threads()
        cpu = {"value": xs.nbytes * len(ts) / sum(ts) / 1e9, "unit": "GB/s", "cores": nth, "kind": "port",
               "sample": f"{len(ts)} full compress(es) of the c5 generator at {CPU_SAMPLE_N}^3 ({xs.nbytes} B, "
                         f"RE {args.re}) via oracle/ (restated reference; Gram and projection loops "
                         f"OpenMP-parallel over {nth} host threads)"}

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(args.re),
        "result": {"input_bytes": nbytes, "ranks": res.ranks, "container_bytes": len(res.container),
                   "compression_factor": res.compression_factor(), "core_last_plane": res.core_last_plane},
        "parallelism": "single GPU",
        "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": len(r2.container),
                "ms_all": [round(v, 2) for v in e2e_ms],
                "python_bytes_ms": round(py_ms, 2),
                "note": "tcb_compress (the C ABI) from pinned host memory (H2D inside), returning with the container "
                        "in host memory (D2H inside); python_bytes_ms: one tcb.compress() that also copies it into a "
                        "Python bytes; "
                        "CUDA events around the synchronous call"},
        "gpu_launches": int(launches),
        "roofline": roof,
        "stage_ms": stage_ms,
        "secondary": secondary,
        "cpu_baseline": cpu,
        "clocks": clk,
        "step_ms_all": [round(v, 3) for v in step_ms],
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
