"""Randomised layer shapes vs the CPU oracle: shard counts 1..16, expert
counts that are not multiples of 16 (the tcgen05 gate pads N), k up to 8,
ragged batches, with / without history, bias, renormalisation.  Seeded, so
a failure names its case."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import layer_ref
from paper_2503_04398_b200 import SpecMoELayer, synth

TOL = 1e-2


def _cases(count=24, seed=None, wide=False):
    """wide: N in 65..256 (the tcgen05 gate's N' = 128 / 160 / 192 / 256
    tournament epilogue); else N <= 64 (register epilogue, split at N' = 64)."""
    import os
    seed = int(os.environ.get("SMOE_FUZZ_SEED", "2025")) if seed is None else seed
    rng = np.random.default_rng(seed + (7919 if wide else 0))
    out = []
    for i in range(count):
        G = int(rng.choice([1, 2, 3, 4, 5, 8, 12, 16]))
        if wide:
            N = int(rng.integers(65, 257))
            N -= N % G                              # clusters of equal size
            N = max(N, 65 + (-65) % G)
        else:
            per = int(rng.integers(1, max(2, 64 // G) + 1))
            N = min(64, G * per)
        k = int(rng.integers(1, min(8, N) + 1))
        d = int(rng.choice([256, 512, 768]))
        f = int(rng.choice([128, 256, 384]))
        n = int(rng.choice([1, 7, 63, 129, 500, 1333, 2100]))
        out.append(dict(i=i, G=G, N=N, k=k, d=d, f=f, n=n, eps=float(rng.uniform(0, 0.8)),
                        hist=bool(rng.random() < 0.7), bias=bool(rng.random() < 0.3),
                        renorm=bool(rng.random() < 0.7)))
    return out


@pytest.mark.parametrize("c", _cases() + _cases(count=10, wide=True),
                         ids=lambda c: "case{i}-G{G}-N{N}-k{k}-d{d}-n{n}".format(**c))
def test_random_layer_matches_oracle(c):
    over = {"G": c["G"], "N": c["N"], "k": c["k"], "d": c["d"], "f": c["f"]}
    w = synth.make_workload("toy", n=c["n"], eps=c["eps"], seed=100 + c["i"], cfg_override=over)
    bias = (np.random.default_rng(c["i"]).normal(scale=0.05, size=c["N"]).astype(np.float32)
            if c["bias"] else None)
    hist = w.hist if c["hist"] else None
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=c["k"],
                         max_tokens=c["n"] + 3, gate_b=bias, renormalize=c["renorm"])
    out = layer.forward(torch.from_numpy(w.partials), w.tokens, hist).float().numpy()
    b = w.bundle
    ref = layer_ref.layer_forward(
        partials=w.partials, tokens=w.tokens, hist=hist, t_labels=b.token_table.labels,
        t_conf=b.token_table.confidence, a_best=b.ngram_table.best,
        a_conf=b.ngram_table.confidence, n_clusters=c["G"], expert_labels=w.expert_labels,
        gate_w=w.gate_w, w1=w.w1, w3=w.w3, w2=w.w2, k=c["k"], renorm=c["renorm"], bias=bias)
    ix = layer.plan_indices(c["n"])
    assert np.array_equal(ix.forward, ref["forward"]) and np.array_equal(ix.inverse, ref["inverse"])
    r = layer.routing(c["n"])
    assert np.array_equal(r["experts"], ref["experts"])
    assert np.allclose(r["weights"], ref["weights"], rtol=1e-4, atol=1e-6)
    st = layer.stats()
    assert (st["local_tokens"], st["remote_tokens"]) == (ref["local"], ref["remote"])
    err = np.linalg.norm(out - ref["out"]) / max(np.linalg.norm(ref["out"]), 1e-30)
    assert err <= TOL, err
