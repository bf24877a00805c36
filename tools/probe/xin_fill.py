"""One forward with the expert-input buffer (xin) pre-filled: stale (torch.empty),
zeros or small noise -- rows of a 128-row A tile past an expert's rows are
whatever the buffer holds, and the MMA rate depends on operand values."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import SpecMoELayer, synth
n, name, fill = int(sys.argv[1]), sys.argv[2], sys.argv[3]
max_tokens = int(sys.argv[4]) if len(sys.argv) > 4 else n
w = synth.make_workload(name, n=n, eps=0.2, seed=0, device=True)
layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"], max_tokens=max_tokens)
layer.partial_views(n).copy_(w.partials)
if fill == "zero":
    layer.xin.zero_(); layer.hmid.zero_()
elif fill == "noise":
    layer.xin.normal_(0, 0.01); layer.hmid.normal_(0, 0.01)
elif fill == "noise_xin":
    layer.xin.normal_(0, 0.01)
elif fill == "noise_hmid":
    layer.hmid.normal_(0, 0.01)
elif fill == "big":
    layer.xin.normal_(0, 100.0); layer.hmid.normal_(0, 100.0)
tok = torch.as_tensor(w.tokens, device="cuda"); hist = torch.as_tensor(w.hist, device="cuda")
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
layer.run_device(tok, hist)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
