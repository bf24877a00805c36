"""Per-stage CUDA-event times with programmatic dependent launch on / off
(SMOE_OPT_PDL toggled in-process, interleaved reps).

    python tools/probe/pdl_stages.py --config mixtral --tokens 16384
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    import numpy as np
    import torch
    from paper_2503_04398_b200 import SpecMoELayer, _native as N, synth
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    lib = N.lib()
    w = synth.make_workload(a.config, n=a.tokens, eps=0.2, seed=0, device=True)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"], max_tokens=a.tokens)
    layer.partial_views(a.tokens).copy_(w.partials)
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    names = ["plan", "srs", "gate", "route", "dispatch", "expert_up", "expert_down", "combine_sag"]
    res = {}
    for rep in range(3):
        for pdl in (0, 1):
            N.check(lib.smoe_set_option(N.OPT_PDL, pdl), "opt")
            for _ in range(3):
                layer.run_device(tok, hist)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                layer.run_device(tok, hist)
            e1.record()
            torch.cuda.synchronize()
            full = e0.elapsed_time(e1) / a.steps
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
                  for _ in range(a.steps)]
            for s in range(a.steps):
                ev[s][0].record()
                for j in range(len(names)):
                    layer.run_device(tok, hist, stages=[j])
                    ev[s][j + 1].record()
            torch.cuda.synchronize()
            st = {nm: float(np.mean([ev[s][j].elapsed_time(ev[s][j + 1]) for s in range(a.steps)]))
                  for j, nm in enumerate(names)}
            res.setdefault(pdl, []).append({"full_ms": full, **st})
    for pdl, v in res.items():
        print(json.dumps({"config": a.config, "tokens": a.tokens, "pdl": pdl,
                          "best_full_ms": min(x["full_ms"] for x in v),
                          "stages_ms_med": {k: float(np.median([x[k] for x in v])) for k in names},
                          "full_reps": [x["full_ms"] for x in v]}), flush=True)


if __name__ == "__main__":
    main()
