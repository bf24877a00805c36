"""Steady-state decode A/B of the narrow GEMM: one layer runs a 16 384-token
batch, then two CUDA graphs of the 64-token forward are captured — narrow
off / on (SMOE_OPT_GEMM_NARROW_MAX_ROWS 0 / 16) — and replayed interleaved."""
import json
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import SpecMoELayer, synth, _native as N

cfg = sys.argv[1]
big = synth.make_workload(cfg, n=16384, eps=0.2, seed=0, device=True)
layer = SpecMoELayer(big.bundle, big.gate_w, big.w1, big.w3, big.w2, top_k=big.cfg["k"],
                     max_tokens=16384)
layer.partial_views(16384).copy_(big.partials)
layer.run_device(torch.as_tensor(big.tokens, device="cuda"), torch.as_tensor(big.hist, device="cuda"))
n = 64
layer.partial_views(n).copy_(big.partials[:, :n])
tok = torch.as_tensor(big.tokens[:n], device="cuda")
hist = torch.as_tensor(big.hist[:n], device="cuda")
lib = N.lib()
graphs, outs = {}, {}
for rows in (0, 16):
    N.check(lib.smoe_set_option(N.OPT_GEMM_NARROW_MAX_ROWS, rows), "opt")
    for _ in range(3):
        layer.run_device(tok, hist)
    graphs[rows] = layer.capture(tok, hist)
    graphs[rows].replay()
    torch.cuda.synchronize()
    outs[rows] = layer.out_view(n).clone()
res = {0: [], 16: []}
for rep in range(6):
    for rows in (0, 16) if rep % 2 == 0 else (16, 0):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(50):
            graphs[rows].replay()
        e1.record()
        torch.cuda.synchronize()
        res[rows].append(round(e0.elapsed_time(e1) / 50 * 1e3, 1))
print(json.dumps({"config": cfg, "us_wide": res[0], "us_narrow": res[16],
                  "median_wide": sorted(res[0])[3], "median_narrow": sorted(res[16])[3],
                  "identical": bool(torch.equal(outs[0], outs[16]))}), flush=True)
