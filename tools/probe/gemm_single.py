"""Standalone grouped GEMM (smoe_grouped_gemm, SwiGLU epilogue) on one or more
problems, cta_group from argv, for ncu DRAM-traffic experiments."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import _native as N
cg, P, M, K, NB = (int(x) for x in sys.argv[1:6])
scale = float(sys.argv[6]) if len(sys.argv) > 6 else 1.0     # B ~ N(0, scale^2)
lib = N.lib()
N.check(lib.smoe_set_option(N.OPT_GEMM_CTA_GROUP_UP, cg), "opt")
A = torch.randn(P * M, K, device="cuda").to(torch.bfloat16)
B = (torch.randn(P * NB, K, device="cuda") * scale).to(torch.bfloat16)
C = torch.empty(P * M, NB // 2, device="cuda", dtype=torch.bfloat16)
probs = torch.tensor([[p * M, M, p, p * M] for p in range(P)], dtype=torch.int64, device="cuda")
def run():
    N.check(lib.smoe_grouped_gemm(N.ptr(A), P * M, K, N.ptr(B), P * NB, NB, N.ptr(probs), P, 1,
                                  N.ptr(C), P * M, NB // 2, N.stream_ptr()), "gemm")
run(); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart(); run(); torch.cuda.synchronize(); torch.cuda.cudart().cudaProfilerStop()
