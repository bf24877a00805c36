"""Interleaved A/B of the expert GEMMs: cta_group::1 vs ::2 on the same
layer, same inputs, alternating reps (so clock / power drift hits both)."""

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main(name="mixtral", tokens=16384, reps=6, steps=5, which="both"):
    import torch
    from paper_2503_04398_b200 import SpecMoELayer, synth
    from paper_2503_04398_b200 import _native as N
    w = synth.make_workload(name, n=tokens, eps=0.2, seed=0, device=True)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"],
                         max_tokens=tokens)
    layer.partial_views(tokens).copy_(w.partials)
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    lib = N.lib()
    layer.run_device(tok, hist)
    res = {1: {"up": [], "down": []}, 2: {"up": [], "down": []}}
    s = torch.cuda.current_stream()
    ref = None
    for rep in range(reps):
        for cg in (1, 2) if rep % 2 == 0 else (2, 1):
            keys = {"both": (N.OPT_GEMM_CTA_GROUP_UP, N.OPT_GEMM_CTA_GROUP_DOWN),
                    "up": (N.OPT_GEMM_CTA_GROUP_UP,),
                    "down": (N.OPT_GEMM_CTA_GROUP_DOWN,)}[which]
            for key in keys:
                N.check(lib.smoe_set_option(key, cg), "set_option")
            layer.run_device(tok, hist)       # warm (maps rebuilt on switch)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            up = dn = 0.0
            for _ in range(steps):
                layer.run_device(tok, hist, stages=range(5))
                ev[0].record(s)
                layer.run_device(tok, hist, stages=[N.STAGE_EXPERT_UP])
                ev[1].record(s)
                layer.run_device(tok, hist, stages=[N.STAGE_EXPERT_DOWN])
                ev[2].record(s)
                layer.run_device(tok, hist, stages=[N.STAGE_COMBINE_SAG])
                torch.cuda.synchronize()
                up += ev[0].elapsed_time(ev[1])
                dn += ev[1].elapsed_time(ev[2])
            res[cg]["up"].append(up / steps)
            res[cg]["down"].append(dn / steps)
            out = layer.out_view(tokens).clone()
            if ref is None:
                ref = out
            if not torch.equal(out, ref):
                print("note: outputs differ, max abs", (out.float() - ref.float()).abs().max().item())
    st = layer.stats(tokens)
    pairs = st["local_tokens"] + st["remote_tokens"]
    d, f = w.cfg["d"], w.cfg["f"]
    for cg in (1, 2):
        up, dn = np.median(res[cg]["up"]), np.median(res[cg]["down"])
        print(json.dumps({"config": name, "tokens": tokens, "cta_group": cg, "which": which,
                          "up_ms": up, "down_ms": dn,
                          "up_tflops": 4.0 * pairs * d * f / up / 1e9,
                          "down_tflops": 2.0 * pairs * d * f / dn / 1e9,
                          "reps_up": res[cg]["up"], "reps_down": res[cg]["down"]}))


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "mixtral", int(a[1]) if len(a) > 1 else 16384,
         reps=int(a[3]) if len(a) > 3 else 6, which=a[2] if len(a) > 2 else "both")
