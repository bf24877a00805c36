"""Standalone down-GEMM-shaped grouped GEMM (store epilogue) at full and half K:
does halving K (what a split-K down GEMM would run per pass) bring DRAM
traffic to the algorithmic bytes at full tensor-pipe occupancy?

    python tools/probe/gemm_splitk_probe.py <cg> <P> <M> <K> <NB>
"""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import _native as N
cg, P, M, K, NB = (int(x) for x in sys.argv[1:6])
lib = N.lib()
N.check(lib.smoe_set_option(N.OPT_GEMM_CTA_GROUP_DOWN, cg), "opt")
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.randn(P * M, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
B = (torch.randn(P * NB, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
C = torch.empty(P * M, NB, device="cuda", dtype=torch.bfloat16)
import os
# SMOE_PROBE_MS="4036,4180,...": per-problem row counts (rows padded to M in A / C)
ms = [int(x) for x in os.environ["SMOE_PROBE_MS"].split(",")] if os.environ.get("SMOE_PROBE_MS") \
    else [M] * P
probs = torch.tensor([[p * M, ms[p], p, p * M] for p in range(P)], dtype=torch.int64,
                     device="cuda")
def run():
    N.check(lib.smoe_grouped_gemm(N.ptr(A), P * M, K, N.ptr(B), P * NB, NB, N.ptr(probs), P, 0,
                                  N.ptr(C), P * M, NB, N.stream_ptr()), "gemm")
for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record()
torch.cuda.synchronize()
ms_ = e0.elapsed_time(e1) / 10
print({"cg": cg, "P": P, "M": M, "K": K, "NB": NB, "ms": round(ms_, 4), "rows": sum(ms),
       "tflops": round(2 * sum(ms) * K * NB / ms_ / 1e9, 1)}, flush=True)
