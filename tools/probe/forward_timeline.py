"""Gantt chart of one decode-sized layer forward (CUDA-graph replay), from
%globaltimer stamps in every layer kernel (instrumented build):

    python -m paper_2503_04398_b200.build --variant tl -DSMOE_TIMELINE
    SMOE_LIB=$PWD/paper_2503_04398_b200/libsmoe_tl.so \
        python tools/probe/forward_timeline.py dsv2_lite 64 [--replays 3]

Per kernel (plan, SRS, gate, dispatch, up GEMM, down GEMM, combine + SAG):
first CTA entry, last CTA past its PDL wait, first / last CTA exit, in us
relative to the plan kernel's entry, for the last of --replays back-to-back
graph replays (steady state: replays overlap only through the stream order).
"""
import argparse
import ctypes as C
import json
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import SpecMoELayer, synth, _native as N  # noqa: E402

KINDS = {0: "plan", 1: "srs", 2: "gate", 4: "dispatch", 5: "expert_up", 6: "expert_down",
         7: "combine_sag"}
UNITS = ("plan", "layer", "gate", "gemm")


def read(lib):
    tot = np.zeros((8, 256, 3), dtype=np.uint64)
    for u in UNITS:
        buf = (C.c_ulonglong * (8 * 256 * 3))()
        assert getattr(lib, f"smoe_probe_tl_{u}")(buf) == 0
        tot = np.maximum(tot, np.frombuffer(buf, dtype=np.uint64).reshape(8, 256, 3))
    return tot.astype(np.int64)


def reset(lib):
    for u in UNITS:
        assert getattr(lib, f"smoe_probe_tl_reset_{u}")() == 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("tokens", type=int)
    ap.add_argument("--replays", type=int, default=3)
    ap.add_argument("--big", type=int, default=2048)
    ap.add_argument("--opt", action="append", default=[], help="KEY=VALUE smoe_set_option")
    a = ap.parse_args()
    for kv in a.opt:
        key, val = (int(x) for x in kv.split("="))
        N.check(N.lib().smoe_set_option(key, val), "set_option")
    n = a.tokens
    big = synth.make_workload(a.config, n=a.big, eps=0.2, seed=0, device=True)
    layer = SpecMoELayer(big.bundle, big.gate_w, big.w1, big.w3, big.w2, top_k=big.cfg["k"],
                         max_tokens=a.big)
    layer.partial_views(a.big).copy_(big.partials)
    layer.run_device(torch.as_tensor(big.tokens, device="cuda"),
                     torch.as_tensor(big.hist, device="cuda"))   # steady-state buffers
    w = synth.make_workload(a.config, n=n, eps=0.2, seed=0, device=True)
    layer.partial_views(n).copy_(w.partials)
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    g = layer.capture(tok, hist)
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    lib = N.lib()
    out = []
    for rep in range(3):
        reset(lib)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for r in range(a.replays):
            if r == a.replays - 1:
                e0.record()
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        tl = read(lib)
        ent = tl[..., 0]
        t0 = ent[0][ent[0] > 0].min()
        rows = {}
        for k, name in KINDS.items():
            m = ent[k] > 0
            if not m.any():
                continue
            e, wt, x = tl[k][m, 0], tl[k][m, 1], tl[k][m, 2]
            rows[name] = {"ctas": int(m.sum()),
                          "entry_first": round((e.min() - t0) / 1e3, 2),
                          "entry_last": round((e.max() - t0) / 1e3, 2),
                          "waited_last": round((wt.max() - t0) / 1e3, 2) if (wt > 0).any() else None,
                          "exit_first": round((x[x > 0].min() - t0) / 1e3, 2) if (x > 0).any() else None,
                          "exit_last": round((x.max() - t0) / 1e3, 2) if (x > 0).any() else None}
        rec = {"config": a.config, "tokens": n, "replay_event_us": round(e0.elapsed_time(e1) * 1e3, 1),
               "kernels": rows}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        for name, r in rows.items():
            print(f"  {name:12s} ctas {r['ctas']:4d}  entry {r['entry_first']:8.2f}..{r['entry_last']:8.2f}"
                  f"  waited {r['waited_last']}  exit {r['exit_first']}..{r['exit_last']}", flush=True)


if __name__ == "__main__":
    main()
