"""Mixtral 16K layer forwards with the up GEMM on cta_group argv[1] (ncu target)."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import SpecMoELayer, synth, _native as N
cg = int(sys.argv[1])
cfg = sys.argv[2] if len(sys.argv) > 2 else "mixtral"
n = 16384
w = synth.make_workload(cfg, n=n, eps=0.2, seed=0, device=True)
layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"], max_tokens=n)
layer.partial_views(n).copy_(w.partials)
tok = torch.as_tensor(w.tokens, device="cuda")
hist = torch.as_tensor(w.hist, device="cuda")
N.check(N.lib().smoe_set_option(N.OPT_GEMM_CTA_GROUP_UP, cg), "opt")
for _ in range(4):
    layer.run_device(tok, hist)
torch.cuda.synchronize()
