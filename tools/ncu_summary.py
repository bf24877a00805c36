"""Summaries of the round-end ncu captures (tools/probe/job_profile.sh):

    python tools/ncu_summary.py launches <launches.csv>   # per-step kernel shares
    python tools/ncu_summary.py full <raw.csv>            # --set full key metrics
"""
import collections
import csv
import sys


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    ii = h.index("ID")
    per = collections.defaultdict(lambda: collections.defaultdict(dict))
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        if not name.startswith("smoe::"):
            continue                      # torch kernels: workload generation
        per[name][r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    t = {k: [m["gpu__time_duration.sum"] / 1e3 for m in v.values()] for k, v in per.items()}
    total = sum(sum(v) for v in t.values())
    dram = any("dram__bytes_read.sum" in m for v in per.values() for m in v.values())
    print("| kernel | launches | mean us | share |" + (" DRAM MB / launch |" if dram else "")
          + "\n|---|---|---|---|" + ("---|" if dram else ""))
    for k, v in per.items():
        line = f"| {k} | {len(t[k])} | {sum(t[k]) / len(t[k]):.1f} | {100 * sum(t[k]) / total:.1f}% |"
        if dram:
            b = [m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
                 for m in v.values()]
            line += f" {sum(b) / len(b) / 1e6:.1f} |"
        print(line)


def full(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    cols = [("time", "gpu__time_duration.sum"), ("dram_read", "dram__bytes_read.sum"),
            ("dram_write", "dram__bytes_write.sum"),
            ("dram_%peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            ("tensor_%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            ("sm_%", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            ("regs", "launch__registers_per_thread"), ("grid", "launch__grid_size"),
            ("sm_clock", "sm__cycles_elapsed.avg.per_second")]
    idx = [h.index(c) for _, c in cols]
    print("| kernel | " + " | ".join(n for n, _ in cols) + " |")
    print("|---" * (len(cols) + 1) + "|")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        vals = [f"{r[i]} {units[i]}".strip() for i in idx]
        print(f"| {name} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
