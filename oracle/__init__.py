"""CPU oracle — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the arithmetic of the reference's online
path (`moesched`, /root/reference/pkg/src/moesched) and the fp32 MoE-layer
formulas the reference does not ship (gate, SwiGLU experts, combine, SRS,
SAG).  It is the checker the parity tests compare
the CUDA path against, and the CPU baseline bench.py times
(`cpu_baseline.kind == "port"`).  Nothing in `paper_2503_04398_b200/` may
import it; the product path fails loudly without libsmoe.so instead.

Parity pinning: `scheduler_ref` is validated against golden vectors produced
by running the reference itself in this container (tests/golden/, generated
by tests/golden/make_golden.py) and against the reference tests' own known
answers.  `layer_ref`'s floating-point half has no reference implementation
(SURVEY.md §8c): it is pinned only by its formulas (stated per function).
"""
