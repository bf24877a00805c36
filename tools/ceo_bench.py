"""§8f rank 4 measurement: one solve_ceo iteration's sample scoring
(solver.py:380-404) on the GPU (smoe_ceo_sample_scores, device-resident
inputs, CUDA events) vs the reference's numpy expression on the host
(one-hot tensordot + reductions, float64), default SolverConfig (K = 64).

    python tools/ceo_bench.py [--tokens 32000] [--experts 64] [--clusters 8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch
    from paper_2503_04398_b200 import _native as N
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=32000)
    ap.add_argument("--experts", type=int, default=64)
    ap.add_argument("--clusters", type=int, default=8)
    ap.add_argument("--samples", type=int, default=64)
    a = ap.parse_args()
    T, Nn, E, K = a.tokens, a.experts, a.clusters, a.samples
    rng = np.random.default_rng(0)
    counts = rng.zipf(1.6, size=(T, Nn)).clip(max=10**6) - 1
    ep = np.stack([rng.permutation(np.arange(Nn) % E) for _ in range(K)])
    tk = rng.integers(0, E, size=(K, T))
    L = N.lib()
    cnt = torch.as_tensor(np.ascontiguousarray(counts.T, dtype=np.int32), device="cuda")
    ep_d = torch.as_tensor(ep.astype(np.int32), device="cuda")
    tk_d = torch.as_tensor(tk.astype(np.int32), device="cuda")
    es = torch.empty(K, dtype=torch.int64, device="cuda")
    js = torch.empty(K, dtype=torch.int64, device="cuda")
    call = lambda: L.smoe_ceo_sample_scores(N.ptr(cnt), T, Nn, N.ptr(ep_d), N.ptr(tk_d), K, E,  # noqa: E731
                                            N.ptr(es), N.ptr(js), N.stream_ptr())
    for _ in range(3):
        N.check(call(), "ceo")
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1) / reps
    # the reference's expressions (solver.py:388-399), float64, on the host
    sub = counts.astype(np.float64)
    t0 = time.perf_counter()
    onehot = np.zeros((K, Nn, E))
    onehot[np.arange(K)[:, None], np.arange(Nn)[None, :], ep] = 1.0
    cm = np.tensordot(sub, onehot, axes=([1], [1])).transpose(1, 0, 2)
    ep_scores = cm.max(axis=2).sum(axis=1)
    joint = cm[np.arange(K)[:, None], np.arange(T)[None, :], tk].sum(axis=1)
    cpu_ms = (time.perf_counter() - t0) * 1e3
    same = bool(np.array_equal(es.cpu().numpy().astype(np.float64), ep_scores) and
                np.array_equal(js.cpu().numpy().astype(np.float64), joint))
    ops = K * T * Nn
    print(json.dumps({"metric": "solve_ceo sample scoring per iteration", "tokens": T,
                      "experts": Nn, "clusters": E, "samples": K, "gpu_ms": gpu_ms,
                      "cpu_numpy_ms": cpu_ms, "cpu_threads": os.cpu_count(),
                      "speedup": cpu_ms / gpu_ms, "bit_identical": same,
                      "count_reads_per_s": ops / (gpu_ms / 1e3)}))


if __name__ == "__main__":
    main()
