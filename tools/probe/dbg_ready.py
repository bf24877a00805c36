import ctypes as C, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import SpecMoELayer, synth, _native as N
w = synth.make_workload("dsv2_lite", n=64, eps=0.2, seed=0, device=True)
layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"], max_tokens=64)
layer.partial_views(64).copy_(w.partials)
tok = torch.as_tensor(w.tokens, device="cuda"); hist = torch.as_tensor(w.hist, device="cuda")
lib = N.lib()
f = lib.smoe_debug_layer_ready
buf = (C.c_int32 * 256)()
layer.run_device(tok, hist, stages=[0,1,2,3,4]); torch.cuda.synchronize()
layer.run_device(tok, hist, stages=[5]); torch.cuda.synchronize()
f(layer._h, buf, 64); print("after up:", list(buf)[:16])
cm = layer.counts_mat.cpu().numpy(); print("rows per expert", cm.sum(0)[:16])
layer.run_device(tok, hist, stages=[6]); torch.cuda.synchronize()
print("err", int(layer.err.item()))
