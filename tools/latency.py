"""Small-batch (decode-regime) layer latency: eager smoe_layer_forward vs the
same forward replayed from a CUDA graph (SpecMoELayer.capture).

    python tools/latency.py [--config mixtral] [--tokens 64,256,1024,4096]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from paper_2503_04398_b200 import SpecMoELayer, synth
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--tokens", default="64,256,1024,4096")
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    for n in [int(x) for x in a.tokens.split(",")]:
        w = synth.make_workload(a.config, n=n, eps=0.2, seed=0, device=True)
        layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"],
                             max_tokens=n)
        layer.partial_views(n).copy_(w.partials)
        tok = torch.as_tensor(w.tokens, device="cuda")
        hist = torch.as_tensor(w.hist, device="cuda")
        for _ in range(3):
            layer.run_device(tok, hist)
        torch.cuda.synchronize()
        ref = layer.out_view(n).clone()

        def timed(fn):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / a.reps * 1e3

        eager = timed(lambda: layer.run_device(tok, hist))
        g = layer.capture(tok, hist)
        g.replay()
        torch.cuda.synchronize()
        same = bool(torch.equal(layer.out_view(n), ref))
        graph = timed(g.replay)
        import hashlib
        import os
        sha = hashlib.sha1(layer.out_view(n).view(torch.int16).cpu().numpy().tobytes()).hexdigest()
        print(json.dumps({"config": a.config, "tokens": n, "eager_us": eager, "graph_us": graph,
                          "graph_output_identical": same, "out_sha1": sha[:16],
                          "env": {k: v for k, v in os.environ.items() if k.startswith("SMOE_")}}),
              flush=True)
        del layer, w, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
