"""Standalone SRS / SAG (smoe_srs / smoe_sag) vs the oracle: SRS rows are
bit-exact (fp32 sum in shard order, one RNE to bf16); SAG is a pure move."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import layer_ref
from paper_2503_04398_b200 import rebatch_tokens
from paper_2503_04398_b200.collectives import shuffled_all_gather, shuffled_reduce_scatter


@pytest.mark.parametrize("n,G,d", [(1, 2, 64), (777, 4, 256), (3000, 8, 512), (5000, 3, 128)])
def test_srs_and_sag_match_oracle(n, G, d):
    rng = np.random.default_rng(n + G)
    devices = rng.integers(0, G, n)
    devices[: min(n, 3)] = 0                               # uneven groups
    parts = [torch.randn(n, d, device="cuda").to(torch.bfloat16) for _ in range(G)]
    tok_s, ix = rebatch_tokens(torch.arange(n, device="cuda"), torch.as_tensor(devices,
                                                                               device="cuda"), G)
    h = shuffled_reduce_scatter(parts, ix)
    fwd = ix.forward.cpu().numpy()
    counts = np.bincount(devices, minlength=G)
    ref = layer_ref.srs(np.stack([p.float().cpu().numpy() for p in parts]), fwd, counts,
                        ix.group_size)
    for g in range(G):
        assert h[g].shape[0] == counts[g]
        assert np.array_equal(h[g].float().cpu().numpy(), ref[g])
    # SAG of the reduced groups restores the original order: row i = sum_r P_r[i]
    outs = shuffled_all_gather(h, ix, n_outs=2)
    full = np.zeros((n, d), np.float32)
    for g in range(G):
        full[fwd[g * ix.group_size: g * ix.group_size + counts[g]]] = ref[g]
    for o in outs:
        assert np.array_equal(o.float().cpu().numpy(), full)
    # a subset of shards (one process's resident range)
    sub = shuffled_reduce_scatter(parts, ix, shards=range(1, G))
    for g, x in zip(range(1, G), sub):
        assert torch.equal(x, h[g])
