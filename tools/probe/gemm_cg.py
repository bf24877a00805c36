"""One forward with the up / down GEMMs on the given cta_groups (argv: up down
config tokens), for ncu A/B of DRAM traffic and clocks."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import SpecMoELayer, synth, _native as N
up, down, name, n = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
w = synth.make_workload(name, n=n, eps=0.2, seed=0, device=True)
layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"], max_tokens=n)
layer.partial_views(n).copy_(w.partials)
lib = N.lib()
N.check(lib.smoe_set_option(N.OPT_GEMM_CTA_GROUP_UP, up), "opt")
N.check(lib.smoe_set_option(N.OPT_GEMM_CTA_GROUP_DOWN, down), "opt")
tok = torch.as_tensor(w.tokens, device="cuda"); hist = torch.as_tensor(w.hist, device="cuda")
for _ in range(2):
    layer.run_device(tok, hist)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
layer.run_device(tok, hist)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
