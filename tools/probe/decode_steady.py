"""Decode after a larger batch on the same layer: the expert-input rows past
each expert's count then hold earlier activations (steady-state serving), not
the zeros of a fresh allocation."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import SpecMoELayer, synth
name, warm = sys.argv[1], int(sys.argv[2])
big = synth.make_workload(name, n=2048, eps=0.2, seed=0, device=True)
layer = SpecMoELayer(big.bundle, big.gate_w, big.w1, big.w3, big.w2, top_k=big.cfg["k"],
                     max_tokens=2048, expert_rows=2048 * big.cfg["k"])
if warm:
    layer.partial_views(2048).copy_(big.partials)
    layer.run_device(torch.as_tensor(big.tokens, device="cuda"), torch.as_tensor(big.hist, device="cuda"))
n = 64
layer.partial_views(n).copy_(big.partials[:, :n])
tok = torch.as_tensor(big.tokens[:n], device="cuda"); hist = torch.as_tensor(big.hist[:n], device="cuda")
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
layer.run_device(tok, hist)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
