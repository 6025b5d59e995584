"""Turn tools/profile_round.sh's gpurun_out/ captures into profiles/ (tracked).

  python tools/summarize_round.py <round-tag>   e.g. r01
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(PROF, exist_ok=True)

def launch_summary(src, dst, header):
    if not os.path.exists(src):
        return
    shutil.copy(src, dst.replace("_summary.txt", ".csv"))
    summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), src],
                          capture_output=True, text=True).stdout
    with open(dst, "w") as f:
        f.write(header)
        f.write(summ)


shutil.copy(os.path.join(OUT, "bench.json"), os.path.join(PROF, f"bench_{tag}_c5_1e-2.json"))
shutil.copy(os.path.join(OUT, "bench_ref.json"), os.path.join(PROF, f"bench_{tag}_reference.json"))
launch_summary(os.path.join(OUT, "launches_bench.csv"), os.path.join(PROF, f"launches_{tag}_bench_summary.txt"),
               "# ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py --steps 2 --warmup 3 "
               "--no-cpu-baseline --no-secondary\n# (cold-cache, serialised launches of every compress the command "
               "runs: 3 warm-up, 2 timed, e2e, profiled, roofline probes)\n")
launch_summary(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"launches_{tag}_c5_1e-2_summary.txt"),
               "# ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none,\n"
               "# tools/c5_once.py 1e-2 (C5_PROFILE=1 C5_ITERS=2): the launches of ONE c5 compress after one\n"
               "# warm-up (cold-cache, serialised: shares, not the overlapped wall time)\n")
# full capture: per-kernel key metrics
rep = os.path.join(OUT, sys.argv[2] if len(sys.argv) > 2 else "full.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
else:  # profile_round.sh already reduced the report to its raw page on the GPU box
    raw = open(rep.replace(".ncu-rep", "_raw.csv")).read()
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
want = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "B",
    "dram__bytes_write.sum": "B",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "%",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "%",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "%",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "%",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "%",
    "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed": "%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "%",
    "launch__grid_size": "",
    "launch__block_size": "",
}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
         "ns": 1e-3, "us": 1, "ms": 1e3}
ki = hdr.index("Kernel Name")
lines = ["# ncu --set full --clock-control none on one c5 compress (tools/profile_round.sh; first launches of each)",
         "# kernel | grid x block | us | DRAM read+write MB | DRAM GB/s | DRAM % elapsed | DMMA pipe % (of active) | "
         "tensor pipe (tcgen05) active % of elapsed | L2 % | SM % | warps active %"]
for r in data:
    name = r[ki].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
    vals = {}
    for m in want:
        if m in hdr:
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                v = float("nan")
            vals[m] = v * scale.get(units[i], 1)
    us = vals["gpu__time_duration.sum"]
    tb = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    lines.append(f"{name:24s} {int(vals['launch__grid_size']):5d} x {int(vals['launch__block_size']):4d} "
                 f"{us:9.1f} {tb / 1e6:9.2f} {tb / us / 1e3:8.1f} "
                 f"{vals.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', float('nan')):6.1f} "
                 f"{vals.get('sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active', float('nan')):6.1f} "
                 f"{vals.get('TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed', float('nan')):6.1f} "
                 f"{vals.get('lts__throughput.avg.pct_of_peak_sustained_elapsed', float('nan')):6.1f} "
                 f"{vals['sm__throughput.avg.pct_of_peak_sustained_elapsed']:6.1f} "
                 f"{vals['sm__warps_active.avg.pct_of_peak_sustained_active']:6.1f}")
with open(os.path.join(PROF, f"ncu_{tag}_{sys.argv[3] if len(sys.argv) > 3 else 'full'}_summary.txt"), "w") as f:
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))
