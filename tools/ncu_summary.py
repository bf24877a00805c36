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
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    per = collections.defaultdict(list)
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        if not name.startswith("smoe::"):
            continue                      # torch kernels: workload generation
        per[name].append(float(r[vi].replace(",", "")) / 1e3)
    total = sum(sum(v) for v in per.values())
    print("| kernel | launches | mean us | share |\n|---|---|---|---|")
    for k, v in per.items():
        print(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / total:.1f}% |")


def full(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    cols = [("time", "gpu__time_duration.sum"), ("dram_read", "dram__bytes_read.sum"),
            ("dram_write", "dram__bytes_write.sum"),
            ("dram_%peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            ("tensor_%", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
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
