"""Interleaved decode-latency A/B of two builds in ONE process is impossible
(one libsmoe per process), so this alternates processes: for each round and
each lib, run tools/latency.py and keep the graph-replay µs.

    python tools/probe/lib_ab.py <libA.so> <libB.so> <config> <tokens> [rounds]
"""
import json
import os
import subprocess
import sys

a, b, cfg, tok = sys.argv[1:5]
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 4
res = {a: [], b: []}
for _ in range(rounds):
    for lib in (a, b):
        env = dict(os.environ, SMOE_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "tools/latency.py", "--config", cfg, "--tokens", tok,
                              "--reps", "100"], capture_output=True, text=True, env=env)
        line = json.loads(out.stdout.strip().splitlines()[-1])
        res[lib].append(round(line["graph_us"], 2))
for lib, v in res.items():
    s = sorted(v)
    print(json.dumps({"lib": os.path.basename(lib), "config": cfg, "tokens": int(tok),
                      "graph_us": v, "median": s[len(s) // 2]}))
