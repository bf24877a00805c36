"""GPU parity of the scheduler API (K1 lookup+plan, K2 gathers, s-EG) against
the numpy oracle and the reference tests' own known answers."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import scheduler_ref as R
from paper_2503_04398_b200 import scheduler as S
from paper_2503_04398_b200.predictor import DeviceNGramTable, TokenDeviceTable


def make_bundle(rng, E, vocab, n=2, nonzero_rows=None):
    labels = rng.integers(0, E, size=vocab)
    conf = rng.random(vocab).astype(np.float32)
    counts = rng.integers(0, 10, size=(E ** n, E))
    if nonzero_rows is not None:
        counts[rng.random(E ** n) > nonzero_rows] = 0
    tot = counts.sum(1, keepdims=True)
    probs = np.divide(counts, tot, out=np.zeros(counts.shape), where=tot > 0)
    tok = TokenDeviceTable(labels=labels, confidence=conf, provenance=np.zeros(vocab, np.uint8),
                           n_clusters=E)
    ng = DeviceNGramTable(n=n, n_clusters=E, probs=probs, counts=counts)
    return S.LookupBundle(token_table=tok, ngram_table=ng, expert_labels=np.arange(2 * E) % E,
                          layers=4)


def oracle_lookup(b, tokens, hist):
    best, conf = R.ngram_best_conf(b.ngram_table.probs)
    return R.lookup_devices(b.token_table.labels, b.token_table.confidence, best, conf,
                            b.token_table.n_clusters, tokens, hist)


@pytest.mark.parametrize("E,vocab,n", [(2, 16, 1), (4, 32, 50), (8, 1000, 4096),
                                       (8, 32000, 70001), (16, 500, 3000)])
def test_lookup_matches_oracle(E, vocab, n):
    rng = np.random.default_rng(E * 1000 + n)
    b = make_bundle(rng, E, vocab, nonzero_rows=0.7)
    tokens = rng.integers(-vocab, vocab, size=n)
    hist = rng.integers(0, E, size=(n, 2))
    assert np.array_equal(S.lookup_devices(b, tokens, hist), oracle_lookup(b, tokens, hist))
    assert np.array_equal(S.lookup_devices(b, tokens, None), oracle_lookup(b, tokens, None))


def test_lookup_confidence_rules():
    # test_scheduler.py:25-40 known answers
    E = 2
    counts = np.zeros((E ** 2, E))
    counts[3] = [1, 9]
    tot = counts.sum(1, keepdims=True)
    probs = np.divide(counts, tot, out=np.zeros(counts.shape), where=tot > 0)
    tok = TokenDeviceTable(labels=[0, 0], confidence=[0.5, 0.95], provenance=[0, 0], n_clusters=E)
    b = S.LookupBundle(token_table=tok, ngram_table=DeviceNGramTable(2, E, probs, counts),
                       expert_labels=[0, 1, 0, 1], layers=4)
    assert S.lookup_device(b, 0, np.array([1, 1])) == (1, "ngram")
    assert S.lookup_device(b, 1, np.array([1, 1])) == (0, "token")
    assert S.lookup_device(b, 0, np.array([0, 0])) == (0, "token")
    assert S.lookup_device(b, 0, None) == (0, "token")


def test_lookup_index_errors():
    rng = np.random.default_rng(0)
    b = make_bundle(rng, 4, 10)
    with pytest.raises(IndexError):
        S.lookup_devices(b, np.array([10]), None)
    with pytest.raises(IndexError):
        S.lookup_devices(b, np.array([1]), np.array([[4, 4, 4]]))   # row 84 >= 16


def test_deferred_errors_for_device_callers():
    """defer_errors(): no per-call error read-back (host sync); the bits
    accumulate on the device and check_errors() raises the same exception
    class the immediate mode would, then clears them."""
    import torch
    rng = np.random.default_rng(3)
    b = make_bundle(rng, 4, 10)
    good = torch.tensor([1, 2, 3], device="cuda")
    bad = torch.tensor([1, 10], device="cuda")           # token id >= vocab
    with S.defer_errors():
        out = S.lookup_devices(b, good, None)
        S.lookup_devices(b, bad, None)                   # no exception here
        assert out.is_cuda and out.shape == (3,)
        with pytest.raises(IndexError):
            S.check_errors()
        S.check_errors()                                 # cleared
        devs = torch.tensor([0, 5, 1], device="cuda")     # device label >= G
        S.rebatch_tokens(good, devs, 4)
        with pytest.raises(S.SchedulerError):
            S.check_errors()
    with pytest.raises(IndexError):                       # immediate mode again
        S.lookup_devices(b, bad, None)


def test_rebatch_golden():
    # test_scheduler.py:57-63 and :66-72
    sh, ix = S.rebatch_tokens(np.array([10, 11, 12, 13, 14]), np.array([1, 0, 1, 1, 0]), 2)
    assert ix.group_size == 3
    assert sh.tolist() == [11, 14, S.PAD_TOKEN, 10, 12, 13]
    assert S.resume_tokens(sh, ix).tolist() == [10, 11, 12, 13, 14]
    sh, ix = S.rebatch_tokens(np.arange(8), np.zeros(8, dtype=int), 4)
    assert len(sh) == 32 and sh[:8].tolist() == list(range(8))
    with pytest.raises(S.SchedulerError):
        S.rebatch_tokens(np.array([1]), np.array([5]), 2)
    with pytest.raises(S.SchedulerError):
        S.rebatch_tokens(np.array([1, 2]), np.array([0]), 2)


@pytest.mark.parametrize("n,G", [(0, 2), (1, 2), (5, 8), (2048, 4), (2049, 3), (4096, 8),
                                 (70000, 8), (100003, 16), (5000, 200)])
def test_rebatch_matches_oracle(n, G):
    rng = np.random.default_rng(n + G)
    tokens = rng.integers(0, 50000, size=n)
    p = rng.dirichlet(np.ones(G) * 0.5)
    devices = rng.choice(G, size=n, p=p)
    sh, ix = S.rebatch_tokens(tokens, devices, G)
    sh_r, fwd, inv, group = R.rebatch_tokens(tokens, devices, G)
    assert ix.group_size == group
    assert np.array_equal(ix.forward, fwd)
    assert np.array_equal(ix.inverse, inv)
    assert np.array_equal(sh, sh_r)
    assert np.array_equal(S.resume_tokens(sh, ix), tokens)


def test_rebatch_dtypes_preserved():
    for dt in (np.int16, np.int32, np.int64, np.float32):
        tokens = np.arange(7).astype(dt)
        sh, ix = S.rebatch_tokens(tokens, np.array([0, 1, 1, 0, 1, 1, 1]), 2)
        sh_r, *_ = R.rebatch_tokens(tokens, np.array([0, 1, 1, 0, 1, 1, 1]), 2)
        assert sh.dtype == dt and np.array_equal(sh, sh_r)


def test_shuffle_roundtrip_criterion7():
    # test_acceptance.py:160-176 (seed 11), 200 of the 1000 batches
    rng = np.random.default_rng(11)
    for _ in range(200):
        n = int(rng.integers(1, 4097))
        G = int(rng.choice([2, 4, 8]))
        tokens = rng.integers(0, 50_000, size=n)
        devices = rng.integers(0, G, size=n)
        sh, idx = S.rebatch_tokens(tokens, devices, G)
        assert sh.size % G == 0
        real = sh.reshape(G, -1) != S.PAD_TOKEN
        assert np.array_equal(real.sum(1), np.bincount(devices, minlength=G))
        assert np.array_equal(S.resume_tokens(sh, idx), tokens)


def test_rebatch_rows_hidden():
    import torch
    rng = np.random.default_rng(3)
    n, d, G = 1000, 512, 8
    x = torch.randn(n, d, dtype=torch.bfloat16, device="cuda")
    devices = rng.integers(0, G, size=n)
    _, ix = S.rebatch_tokens(np.arange(n), devices, G)
    y = S.rebatch_rows(x, ix)
    fwd = torch.as_tensor(ix.forward, device="cuda")
    ref = torch.where((fwd >= 0)[:, None], x[fwd.clamp(min=0)], torch.zeros_like(x[:1]))
    assert torch.equal(y, ref)
    back = S.resume_tokens(y, ix)
    assert torch.equal(back, x)


def test_gate_permutation_golden_and_random():
    p = S.gate_permutation(np.array([0, 0, 1, 1]), 2)
    assert p.new_to_old.tolist() == [0, 1, 2, 3]
    p = S.gate_permutation(np.array([1, 1, 0, 0]), 2)
    assert p.new_to_old.tolist() == [2, 3, 0, 1]
    rng = np.random.default_rng(13)
    for N, E in ((16, 4), (64, 8), (160, 8)):
        labels = rng.permutation(np.arange(N) % E)
        p = S.gate_permutation(labels, E)
        n2o, o2n = R.gate_permutation(labels, E)
        assert np.array_equal(p.new_to_old, n2o) and np.array_equal(p.old_to_new, o2n)
        logits = rng.normal(size=(5, N))
        assert np.array_equal(S.apply_expert_shuffle(logits, p), R.apply_expert_shuffle(logits, n2o))
        topk = rng.integers(0, N, size=(7, 3))
        assert np.array_equal(S.remap_topk(topk, p), R.remap_topk(topk, o2n))
    with pytest.raises(S.SchedulerError):
        S.gate_permutation(np.array([0, 3]), 2)
    with pytest.raises(S.SchedulerError):
        S.apply_expert_shuffle(np.zeros(3), S.gate_permutation(np.array([0, 1]), 2))


def test_gate_transparency_criterion8():
    # test_acceptance.py:179-193 (seed 13)
    rng = np.random.default_rng(13)
    N, E = 16, 4
    for _ in range(200):
        logits = rng.normal(size=N)
        labels = rng.permutation(np.repeat(np.arange(E), N // E))
        perm = S.gate_permutation(labels, E)
        sh = S.apply_expert_shuffle(logits, perm)
        for k in (1, 2, 6):
            want = set(np.argsort(-logits, kind="stable")[:k])
            got = set(perm.new_to_old[np.argsort(-sh, kind="stable")[:k]])
            assert got == want


def test_schedule_requests_dp_known_answers_and_oracle():
    # test_scheduler.py:125-139 and test_acceptance.py:196-209 (seed 17)
    rng = np.random.default_rng(7)
    E, K = 4, 400
    aff = rng.random((K, E))
    labels = S.schedule_requests_dp(np.ones(K), aff, E)
    for w in range(0, K, E):
        assert sorted(labels[w:w + E].tolist()) == list(range(E))
    a2 = np.zeros((8, 4))
    a2[np.arange(8), np.arange(8) % 4] = 1.0
    assert S.schedule_requests_dp(np.ones(8), a2, 4).tolist() == [0, 1, 2, 3, 0, 1, 2, 3]
    rng = np.random.default_rng(17)
    E, K = 4, 10_000
    preferred = rng.integers(0, E, size=K)
    affinities = rng.random((K, E)) * 0.5
    affinities[np.arange(K), preferred] += 1.0
    labels = S.schedule_requests_dp(rng.integers(1, 512, size=K), affinities, E)
    windows = labels.reshape(-1, E)
    assert np.all(np.sort(windows, axis=1) == np.arange(E))
    assert (windows[:, 0] == preferred[::E]).mean() >= (E - 1) / E
    # vs a direct restatement, ragged last window, ties, G = 7
    for G, K in ((7, 1000), (8, 13), (3, 1)):
        aff = np.round(rng.random((K, G)), 1)          # many ties -> first max wins
        want = np.empty(K, dtype=np.int64)
        for r in range(K):
            if r % G == 0:
                open_ = np.ones(G, bool)
            d = int(np.where(open_, aff[r], -np.inf).argmax())
            want[r] = d
            open_[d] = False
        assert np.array_equal(S.schedule_requests_dp(np.ones(K), aff, G), want)
    with pytest.raises(S.SchedulerError):
        S.schedule_requests_dp(np.ones(3), np.zeros((3, 2)), 4)
