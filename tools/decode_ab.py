"""Interleaved A/B of a layer option at decode-sized batches (CUDA-graph replay).

    python tools/decode_ab.py --config dsv2_lite --tokens 64 --opt 8=0,32,64,96 [--reps 30 --rounds 5]

The layer first runs a 2048-token batch (steady-state serving: the expert
input rows past each expert's count hold earlier activations), then one graph
is captured per option value (the option is read at launch time, i.e. at
capture) and the graphs are replayed in interleaved rounds; prints one JSON
line per value with the median per-round µs and whether its output equals the
first value's bit for bit.
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2503_04398_b200 import SpecMoELayer, synth
    from paper_2503_04398_b200 import _native as N
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="dsv2_lite")
    ap.add_argument("--tokens", type=int, default=64)
    ap.add_argument("--opt", required=True, help="KEY=v1,v2,... (smoe_set_option key)")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--rounds", type=int, default=7)
    ap.add_argument("--big", type=int, default=2048)
    a = ap.parse_args()
    key, vals = a.opt.split("=")
    key, vals = int(key), [int(v) for v in vals.split(",")]
    big = synth.make_workload(a.config, n=a.big, eps=0.2, seed=0, device=True)
    layer = SpecMoELayer(big.bundle, big.gate_w, big.w1, big.w3, big.w2, top_k=big.cfg["k"],
                         max_tokens=a.big)
    lib = layer.lib
    old = lib.smoe_get_option(key)
    layer.partial_views(a.big).copy_(big.partials)
    layer.run_device(torch.as_tensor(big.tokens, device="cuda"),
                     torch.as_tensor(big.hist, device="cuda"))
    n = a.tokens
    layer.partial_views(n).copy_(big.partials[:, :n])
    tok = torch.as_tensor(big.tokens[:n], device="cuda")
    hist = torch.as_tensor(big.hist[:n], device="cuda")
    graphs, outs = [], []
    for v in vals:
        assert lib.smoe_set_option(key, v) == 0, (key, v)
        g = layer.capture(tok, hist)
        g.replay()
        torch.cuda.synchronize()
        outs.append(layer.out_view(n).clone())
        graphs.append(g)
    lib.smoe_set_option(key, old)
    times = [[] for _ in vals]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(a.rounds):
        order = list(range(len(graphs)))
        if r % 2:
            order.reverse()                 # ABBA...: cancels drift within a round
        for i in order:
            g = graphs[i]
            for _ in range(3):
                g.replay()
            e0.record()
            for _ in range(a.reps):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            times[i].append(e0.elapsed_time(e1) / a.reps * 1e3)
    for i, v in enumerate(vals):
        print(json.dumps({"config": a.config, "tokens": n, "opt": key, "value": v,
                          "median_us": statistics.median(times[i]),
                          "min_us": min(times[i]), "rounds_us": [round(x, 1) for x in times[i]],
                          "identical_to_first": bool(torch.equal(outs[i], outs[0]))}), flush=True)


if __name__ == "__main__":
    main()
