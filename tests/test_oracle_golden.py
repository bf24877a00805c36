"""The CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py) and the reference tests' own known answers.
Pins the oracle before it is trusted as the GPU checker."""

import numpy as np
import pytest

from golden_util import cases
from oracle import layer_ref, scheduler_ref as R


@pytest.mark.parametrize("c", cases("lookup"), ids=lambda c: f"E{int(c['E'])}")
def test_lookup_golden(c):
    best, conf = R.ngram_best_conf(c["probs"])
    E = int(c["E"])
    got = R.lookup_devices(c["labels"], c["conf"], best, conf, E, c["tokens"], c["hist"])
    assert np.array_equal(got, c["dev_hist"])
    got = R.lookup_devices(c["labels"], c["conf"], best, conf, E, c["tokens"], None)
    assert np.array_equal(got, c["dev_static"])


@pytest.mark.parametrize("c", cases("rebatch"), ids=lambda c: f"n{len(c['tokens'])}G{int(c['G'])}")
def test_rebatch_golden(c):
    sh, fwd, inv, group = R.rebatch_tokens(c["tokens"], c["devices"], int(c["G"]))
    assert group == int(c["group"])
    assert np.array_equal(fwd, c["forward"]) and np.array_equal(inv, c["inverse"])
    assert np.array_equal(sh, c["shuffled"])
    assert np.array_equal(R.resume(sh, inv), c["resumed"])


def test_rebatch_known_answers():
    # test_scheduler.py:57-72
    sh, fwd, inv, group = R.rebatch_tokens(np.array([10, 11, 12, 13, 14]),
                                           np.array([1, 0, 1, 1, 0]), 2)
    assert group == 3 and sh.tolist() == [11, 14, -1, 10, 12, 13]
    sh, *_ = R.rebatch_tokens(np.arange(8), np.zeros(8, dtype=int), 4)
    assert len(sh) == 32 and sh[:8].tolist() == list(range(8))
    with pytest.raises(R.OracleError):
        R.rebatch_tokens(np.array([1]), np.array([5]), 2)


@pytest.mark.parametrize("c", cases("gate"), ids=lambda c: f"N{len(c['labels'])}")
def test_gate_golden(c):
    n2o, o2n = R.gate_permutation(c["labels"], int(c["E"]))
    assert np.array_equal(n2o, c["new_to_old"]) and np.array_equal(o2n, c["old_to_new"])
    assert np.array_equal(R.apply_expert_shuffle(c["logits"], n2o), c["shuffled"])
    assert np.array_equal(R.remap_topk(c["topk"], o2n), c["remapped"])


@pytest.mark.parametrize("c", cases("simulate"), ids=["planted", "planted_noisy"])
def test_simulate_counts_golden(c):
    E, N = 4, 16
    for i in range(len(c["local"])):
        mode = ("ds_moe", "s_ts", "s_ts_eg")[int(c["mode"][i])]
        loc, rem = R.simulate_counts(c["tokens"], c["routed"][:, int(c["layer"][i]), :], mode, E,
                                     N, c["token_labels"], c["expert_labels"], c["train_counts"])
        assert (loc, rem) == (int(c["local"][i]), int(c["remote"][i]))


@pytest.mark.parametrize("ci", range(3))
def test_toy_lar_known_answers(ci):
    """SURVEY.md §8c toy known answers, recomputed by the oracle."""
    c = cases("toy")[ci]
    want = {0: (0.4875, 0.625, 1.0), 1: (0.4979, 0.6096, 0.7879), 2: (0.5029, 0.5817, 0.6502)}[ci]
    lar = []
    for mode in ("ds_moe", "s_ts", "s_ts_eg"):
        loc = tot = 0
        for layer in range(c["routed"].shape[1]):
            l, r = R.simulate_counts(c["tokens"], c["routed"][:, layer, :], mode, 2, 8,
                                     c["token_labels"], c["expert_labels"], c["train_counts"])
            loc += l
            tot += l + r
        lar.append(loc / tot)
    assert np.allclose(lar, c["lar"], atol=0)
    assert np.allclose(lar, want, atol=5e-5)


def test_bf16_rounding_matches_torch():
    import torch
    x = np.random.default_rng(0).standard_normal(100_000).astype(np.float32) * 100
    x[:4] = [1.00390625, 1.01171875, -2.0078125, 3.0e38]      # ties / large values
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(layer_ref.bf16(x), ref)


def test_layer_oracle_identities():
    """Routing of the oracle reproduces the synthetic generator's planted
    choices (margin construction) and the SRS reduces the partials."""
    from paper_2503_04398_b200 import synth
    w = synth.make_workload("toy", n=200, eps=0.3, seed=3, cfg_override={"G": 4, "N": 16})
    b = w.bundle
    ref = layer_ref.layer_forward(partials=w.partials, tokens=w.tokens, hist=w.hist,
                                  t_labels=b.token_table.labels, t_conf=b.token_table.confidence,
                                  a_best=b.ngram_table.best, a_conf=b.ngram_table.confidence,
                                  n_clusters=4, expert_labels=w.expert_labels, gate_w=w.gate_w,
                                  w1=w.w1, w3=w.w3, w2=w.w2, k=2)
    assert np.array_equal(ref["experts"], w.chosen)
    assert np.allclose(ref["h"], w.partials.sum(0), atol=0.05)
    assert ref["local"] + ref["remote"] == 200 * 2
