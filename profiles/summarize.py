"""Summarise ncu reports / launch lists into the tracked profiles/ directory.

    python profiles/summarize.py gpurun_out/gemm_r1.ncu-rep [...] > profiles/x.md
    python profiles/summarize.py --launches gpurun_out/launches_r1.csv
"""

import csv
import io
import subprocess
import sys
from collections import OrderedDict

METRICS = OrderedDict([
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
])


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"### {path}\n")
    print("| kernel | " + " | ".join(METRICS.values()) + " |")
    print("|---|" + "---|" * len(METRICS))
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        cells = []
        for m in METRICS:
            cells.append(f"{d.get(m, '')} {u.get(m, '')}".strip())
        name = d.get("Kernel Name", "?").split("(")[0]
        print(f"| {name} | " + " | ".join(cells) + " |")
    print()


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0]
            agg.setdefault(name, []).append(float(d["Metric Value"]))
    total = sum(sum(v) for v in agg.values())
    print(f"### launch list {path} (ncu gpu__time_duration, cold-cache, serialised)\n")
    print("| kernel | launches | mean us | share of step |")
    print("|---|---|---|---|")
    for k, v in agg.items():
        print(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / total:.1f}% |")
    print()


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--launches":
        for p in args[1:]:
            launches(p)
    else:
        for p in args:
            report(p)
