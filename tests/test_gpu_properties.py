"""Property tests (hypothesis) of the GPU scheduler mirror, after the
reference's own properties (test_scheduler.py:75-84 round trip, :103-114
top-k invariance under the s-EG gate permutation), plus batch-level
properties of the plan the reference states in rebatch_tokens' docstring."""

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

pytestmark = pytest.mark.gpu

from paper_2503_04398_b200 import scheduler as S


@settings(max_examples=200, deadline=None)
@given(st.integers(1, 3000), st.sampled_from([1, 2, 3, 4, 8, 16]), st.integers(0, 2 ** 31 - 1))
def test_rebatch_resume_roundtrip_and_stability(n, G, seed):
    rng = np.random.default_rng(seed)
    tokens = rng.integers(0, 100_000, size=n)
    devices = rng.integers(0, G, size=n)
    shuffled, ix = S.rebatch_tokens(tokens, devices, G)
    assert len(shuffled) == G * ix.group_size
    assert ix.group_size == np.bincount(devices, minlength=G).max()
    assert np.array_equal(S.resume_tokens(shuffled, ix), tokens)
    fwd = np.asarray(ix.forward).reshape(G, -1)
    for g in range(G):                         # stable, device-contiguous, pads last
        real = fwd[g][fwd[g] >= 0]
        assert np.all(np.diff(real) > 0) and np.all(devices[real] == g)
        assert np.all(fwd[g][len(real):] == -1)


@settings(max_examples=200, deadline=None)
@given(st.integers(0, 2 ** 31 - 1), st.sampled_from([1, 2, 6]), st.sampled_from([(16, 4), (64, 8)]))
def test_gate_shuffle_keeps_topk(seed, k, shape):
    N, E = shape
    rng = np.random.default_rng(seed)
    labels = rng.permutation(np.arange(N) % E)
    perm = S.gate_permutation(labels, E)
    logits = rng.normal(size=(3, N))
    shuffled = np.asarray(S.apply_expert_shuffle(logits, perm))
    n2o = np.asarray(perm.new_to_old)
    for r in range(3):
        orig = set(np.argsort(-logits[r], kind="stable")[:k].tolist())
        new = n2o[np.argsort(-shuffled[r], kind="stable")[:k]]
        assert set(new.tolist()) == orig
    # remap_topk maps original expert ids to their s-EG slots (old_to_new,
    # scheduler.py:222-224): the original top-k lands on the shuffled top-k
    orig_top = np.argsort(-logits, axis=1, kind="stable")[:, :k]
    slot_top = np.argsort(-shuffled, axis=1, kind="stable")[:, :k]
    assert np.array_equal(np.asarray(S.remap_topk(orig_top, perm)), slot_top)
