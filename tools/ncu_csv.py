"""Pretty-print an ncu --csv metrics log: one line per kernel launch."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
out = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"].split("(")[0])
        out.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"]
for (i, name), m in out.items():
    print(i, name, {k: v for k, v in m.items()})
