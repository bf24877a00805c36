"""§8f rank 4: solve_ceo's sample scoring on the GPU (smoe_ceo_sample_scores)
vs the reference's own values (tests/golden/ceo.npz) and the oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from golden_util import cases
from oracle import solver_ref
from paper_2503_04398_b200 import ceo_sample_scores
from paper_2503_04398_b200.solver import SolverError


@pytest.mark.parametrize("c", cases("ceo"), ids=lambda c: f"t{c['counts'].shape[0]}")
def test_ceo_scores_match_reference(c):
    ep_s, tk_s, joint = ceo_sample_scores(c["counts"], c["ep"], c["tk"], c["p_ep"])
    assert np.array_equal(ep_s, c["ep_scores"])
    assert np.array_equal(joint, c["joint"])
    assert np.array_equal(tk_s, c["tk_scores"])


@pytest.mark.parametrize("T,N,E,K", [(32000, 64, 8, 64), (5000, 8, 2, 20), (777, 24, 3, 9),
                                     (1, 4, 2, 1)])
def test_ceo_scores_large_vs_oracle(T, N, E, K):
    """Vocabulary-sized inputs (Mixtral vocab, N = 64 experts, K = 64 samples,
    the default SolverConfig) with heavy-tailed counts, and ragged shapes."""
    rng = np.random.default_rng(T + N)
    counts = rng.zipf(1.6, size=(T, N)).clip(max=10**6) - 1
    ep = np.stack([rng.permutation(np.arange(N) % E) for _ in range(K)])
    tk = rng.integers(0, E, size=(K, T))
    got = ceo_sample_scores(counts, ep, tk)
    want = solver_ref.ceo_scores(counts, ep, tk)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[2], want[2])
    assert got[1] is None


def test_ceo_scores_edge_cases():
    assert [len(x) for x in ceo_sample_scores(np.zeros((5, 4), np.int64),
                                              np.zeros((0, 4)), np.zeros((0, 5)))[::2]] == [0, 0]
    ep_s, _, joint = ceo_sample_scores(np.zeros((3, 4), np.int64), np.zeros((2, 4), np.int64),
                                       np.zeros((2, 3), np.int64))
    assert not ep_s.any() and not joint.any()
    with pytest.raises(SolverError):
        ceo_sample_scores(np.zeros((3, 4)), np.zeros((2, 5)), np.zeros((2, 3)))
    with pytest.raises(SolverError):
        ceo_sample_scores(-np.ones((3, 4)), np.zeros((2, 4)), np.zeros((2, 3)))
