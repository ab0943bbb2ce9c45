"""Summarise ncu outputs into profiles/: key metrics of a --set full capture
(per kernel) and the share of each kernel in a launch list.

    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep profiles/rNN_x.txt
    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/rNN_launches.txt
"""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__grid_size",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes.sum.per_second",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__average_warp_latency_per_inst_issued.ratio",
    "smsp__inst_executed.sum",
]
STALLS = "smsp__average_warps_issue_stalled_"


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    hdr, units = rows[0], rows[1]
    with open(out, "w") as f:
        for row in rows[2:]:
            d = dict(zip(hdr, row))
            f.write(f"== {d.get('Kernel Name', '?')[:160]}\n")
            for k in KEYS:
                if k in d:
                    f.write(f"  {k} = {d[k]} {units[hdr.index(k)]}\n")
            for k in hdr:
                if k.startswith(STALLS) and k.endswith("_per_issue_active.ratio"):
                    try:
                        v = float(d[k])
                    except ValueError:
                        continue
                    if v >= 0.02:
                        name = k[len(STALLS):-len("_per_issue_active.ratio")]
                        f.write(f"  stall {name} = {v:.3f}\n")


def launches(csv_path, out):
    lines = open(csv_path).read().splitlines()
    start = next(i for i, line in enumerate(lines) if line.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][:110]
        v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
        tot[name] += v
        cnt[name] += 1
    allt = sum(tot.values())
    with open(out, "w") as f:
        f.write(f"{'share':>7} {'launches':>8} {'total_ms':>12}  kernel\n")
        for k in sorted(tot, key=tot.get, reverse=True):
            f.write(f"{100 * tot[k] / allt:6.2f}% {cnt[k]:8d} {tot[k] / 1e6:12.3f}  {k}\n")


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    (full if mode == "full" else launches)(src, dst)
