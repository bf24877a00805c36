import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import SpecMoELayer, synth
n = int(sys.argv[1]); name = sys.argv[2]
w = synth.make_workload(name, n=n, eps=0.2, seed=0, device=True)
layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"], max_tokens=n)
layer.partial_views(n).copy_(w.partials)
tok = torch.as_tensor(w.tokens, device="cuda"); hist = torch.as_tensor(w.hist, device="cuda")
for _ in range(5): layer.run_device(tok, hist)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): layer.run_device(tok, hist)
e1.record(); torch.cuda.synchronize()
print("fwd_us", e0.elapsed_time(e1) / 20 * 1e3)
torch.cuda.cudart().cudaProfilerStart()
layer.run_device(tok, hist)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
