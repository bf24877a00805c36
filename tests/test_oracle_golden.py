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


# ---------------------------------------------------------------- round 2 pins
@pytest.mark.parametrize("c", cases("metrics"), ids=lambda c: "trace" if int(c["kind"]) else "matrix")
def test_metrics_golden(c):
    """solver.metrics (solver.py:766-800) restated; golden values from the
    reference on its planted fixtures (truth / round-robin / solved)."""
    if int(c["kind"]):
        m = layer_ref.metrics(c["token_labels"], c["expert_labels"], tokens=c["tokens"],
                              routed=c["routed"])
    else:
        m = layer_ref.metrics(c["token_labels"], c["expert_labels"], counts=c["counts"])
    assert m["lar"] == float(c["lar"]) and m["imbalance"] == float(c["imbalance"])
    assert m["events"] == int(c["events"]) and m["local_events"] == int(c["local_events"])


def test_metrics_known_answer_truth():
    # test_solver.py:342-351: truth assignment -> LAR 1.0, imbalance 1.0,
    # events = k * L * occurrences
    c = cases("metrics")[0]
    m = layer_ref.metrics(c["token_labels"], c["expert_labels"], tokens=c["tokens"],
                          routed=c["routed"])
    assert m["lar"] == 1.0 and m["imbalance"] == 1.0
    assert m["events"] == 2 * 3 * len(c["tokens"])


def _chain(ci):
    from golden_util import toy_bundle_path
    from paper_2503_04398_b200 import tables
    b = tables.read_bundle(toy_bundle_path(ci))
    return b, cases("toy")[ci], cases("toy_chain")[ci]


@pytest.mark.parametrize("ci", range(3))
def test_toy_chain_oracle(ci):
    """configs[0] three-layer chain: the oracle's lookup with the history
    window it builds itself (next_window, depth-tracked: T-only until two
    layers were observed) equals the reference's per-layer lookup / plan /
    local events (tests/golden/toy_chain.npz)."""
    b, toy, ch = _chain(ci)
    tokens, routed = toy["tokens"], toy["routed"]
    C = np.asarray(b.expert_labels, dtype=np.int64)
    best, conf = R.ngram_best_conf(b.ngram_table.probs)
    win, depth = None, 0
    for layer in range(3):
        lookup_hist = win if (win is not None and depth >= 2) else None
        dev = R.lookup_devices(b.token_table.labels, b.token_table.confidence, best, conf, 2,
                               tokens, lookup_hist)
        pre = f"l{layer}_"
        assert np.array_equal(dev, ch[pre + "dev"])
        if lookup_hist is not None:
            assert np.array_equal(lookup_hist, ch[pre + "hist"])
        sh, fwd, inv, group = R.rebatch_tokens(tokens, dev, 2)
        assert np.array_equal(fwd, ch[pre + "forward"]) and group == int(ch[pre + "group"])
        assert R.count_local(routed[:, layer], C, dev) == int(ch[pre + "local"])
        win, depth = layer_ref.next_window(win, depth, C[routed[:, layer, 0]], 2)


def test_gate_topk_slot_space_ties():
    """Ties are broken in s-EG slot space (test_acceptance.py:179-193): the
    first k of a stable argsort of the SHUFFLED logits, remapped; -inf logits
    remain candidates, so fewer than k finite logits still yield k experts."""
    labels = np.array([1, 0, 1, 0])             # slot order: experts 1, 3, 0, 2
    n2o, _ = R.gate_permutation(labels, 2)
    assert n2o.tolist() == [1, 3, 0, 2]
    logits = np.array([[1.0, 1.0, 0.0, 0.0],    # 0 and 1 tie: expert 1 (slot 0) before 0 (slot 2)
                       [0.0, 2.0, 0.0, 2.0],    # 1 and 3 tie: expert 1 (slot 0) first
                       [-np.inf, -np.inf, 5.0, -np.inf],
                       [-np.inf] * 4])
    ids, w, _ = layer_ref.gate_topk(None, None, 2, True, new_to_old=n2o, logits=logits)
    assert ids[0].tolist() == [1, 0] and ids[1].tolist() == [1, 3]
    assert ids[2].tolist() == [2, 1]            # finite first, then the lowest -inf SLOT
    assert ids[3].tolist() == [1, 3]
    assert w[2].tolist() == [1.0, 0.0]
    # identity slot order = the reference's argsort over original ids
    ids, _, _ = layer_ref.gate_topk(None, None, 2, True, logits=logits)
    assert ids[0].tolist() == [0, 1] and ids[2].tolist() == [2, 0]


@pytest.mark.parametrize("c", cases("ceo"), ids=lambda c: f"t{c['counts'].shape[0]}")
def test_ceo_scores_golden(c):
    """oracle.solver_ref vs the reference's solve_ceo scoring expressions and
    its `_sample_scores` (tests/golden/ceo.npz), bit for bit."""
    from oracle import solver_ref
    ep_s, tk_s, joint = solver_ref.ceo_scores(c["counts"], c["ep"], c["tk"], c["p_ep"])
    assert np.array_equal(ep_s, c["ep_scores"])
    assert np.array_equal(joint, c["joint"])
    assert np.array_equal(tk_s, c["tk_scores"])
