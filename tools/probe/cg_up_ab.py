"""Interleaved A/B of the up GEMM's cta_group (1: one SM per 128x256 tile,
2: SM pair per 256x256 tile) inside the full layer at full size: ABBA rounds
of whole-forward timing plus the up-GEMM stage alone.

    python tools/probe/cg_up_ab.py [config] [tokens] [rounds]
"""
import json
import statistics
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import SpecMoELayer, synth, _native as N

cfg = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 6
w = synth.make_workload(cfg, n=n, eps=0.2, seed=0, device=True)
layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"], max_tokens=n)
layer.partial_views(n).copy_(w.partials)
tok = torch.as_tensor(w.tokens, device="cuda")
hist = torch.as_tensor(w.hist, device="cuda")
lib = N.lib()
old = lib.smoe_get_option(N.OPT_GEMM_CTA_GROUP_UP)
up = N.STAGE_NAMES.index("expert_up")
res = {1: {"step": [], "up": []}, 2: {"step": [], "up": []}}
outs = {}
try:
    for cg in (1, 2):
        N.check(lib.smoe_set_option(N.OPT_GEMM_CTA_GROUP_UP, cg), "opt")
        for _ in range(3):
            layer.run_device(tok, hist)
        torch.cuda.synchronize()
        outs[cg] = layer.out_view(n).clone()
    for r in range(rounds):
        for cg in ((1, 2) if r % 2 == 0 else (2, 1)):
            N.check(lib.smoe_set_option(N.OPT_GEMM_CTA_GROUP_UP, cg), "opt")
            layer.run_device(tok, hist)
            e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
            torch.cuda.synchronize()
            e0.record()
            for _ in range(5):
                layer.run_device(tok, hist)
            e1.record()
            layer.run_device(tok, hist, stages=list(range(up)))
            e2.record()
            layer.run_device(tok, hist, stages=[up])
            e3.record()
            layer.run_device(tok, hist, stages=list(range(up + 1, len(N.STAGE_NAMES))))
            torch.cuda.synchronize()
            res[cg]["step"].append(e0.elapsed_time(e1) / 5)
            res[cg]["up"].append(e2.elapsed_time(e3))
finally:
    N.check(lib.smoe_set_option(N.OPT_GEMM_CTA_GROUP_UP, old), "opt")
print(json.dumps({"config": cfg, "tokens": n, "identical": bool(torch.equal(outs[1], outs[2])),
                  "cg1_step_ms": statistics.median(res[1]["step"]),
                  "cg2_step_ms": statistics.median(res[2]["step"]),
                  "cg1_up_ms": statistics.median(res[1]["up"]),
                  "cg2_up_ms": statistics.median(res[2]["up"]),
                  "rounds": {k: {kk: [round(x, 3) for x in vv] for kk, vv in v.items()}
                             for k, v in res.items()}}), flush=True)
