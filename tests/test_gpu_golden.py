"""CUDA path against the golden vectors the reference itself produced."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from golden_util import cases, toy_bundle_path
from paper_2503_04398_b200 import comm, scheduler as S, tables
from paper_2503_04398_b200.predictor import DeviceNGramTable, TokenDeviceTable


def bundle_of(c):
    E = int(c["E"])
    tok = TokenDeviceTable(labels=c["labels"], confidence=c["conf"],
                           provenance=np.zeros(len(c["labels"]), np.uint8), n_clusters=E)
    ng = DeviceNGramTable(n=2, n_clusters=E, probs=c["probs"], counts=c["counts"])
    return S.LookupBundle(token_table=tok, ngram_table=ng, expert_labels=np.arange(2 * E) % E,
                          layers=4)


@pytest.mark.parametrize("c", cases("lookup"), ids=lambda c: f"E{int(c['E'])}")
def test_lookup_golden(c):
    b = bundle_of(c)
    assert np.array_equal(S.lookup_devices(b, c["tokens"], c["hist"]), c["dev_hist"])
    assert np.array_equal(S.lookup_devices(b, c["tokens"], None), c["dev_static"])
    for i in range(len(c["scalar_dev"])):
        dev, src = S.lookup_device(b, int(c["tokens"][i]), c["hist"][i])
        assert dev == int(c["scalar_dev"][i])
        assert (src == "ngram") == bool(c["scalar_ngram"][i])


@pytest.mark.parametrize("c", cases("rebatch"), ids=lambda c: f"n{len(c['tokens'])}G{int(c['G'])}")
def test_rebatch_golden(c):
    sh, ix = S.rebatch_tokens(c["tokens"], c["devices"], int(c["G"]))
    assert ix.group_size == int(c["group"])
    assert np.array_equal(ix.forward, c["forward"]) and np.array_equal(ix.inverse, c["inverse"])
    assert np.array_equal(sh, c["shuffled"]) and sh.dtype == c["shuffled"].dtype
    assert np.array_equal(S.resume_tokens(sh, ix), c["resumed"])


@pytest.mark.parametrize("c", cases("gate"), ids=lambda c: f"N{len(c['labels'])}")
def test_gate_golden(c):
    p = S.gate_permutation(c["labels"], int(c["E"]))
    assert np.array_equal(p.new_to_old, c["new_to_old"])
    assert np.array_equal(p.old_to_new, c["old_to_new"])
    sh = S.apply_expert_shuffle(c["logits"], p)
    assert sh.dtype == c["shuffled"].dtype and np.array_equal(sh, c["shuffled"])
    assert np.array_equal(S.remap_topk(c["topk"], p), c["remapped"])


class _Trace:
    def __init__(self, tokens, routed):
        self._t, self._r = tokens, routed

    def all_tokens(self):
        return self._t

    def all_routed(self):
        return self._r


class _Topo:
    def __init__(self, E, N, k):
        self.clusters, self.experts, self.top_k = E, N, k
        self.experts_per_cluster = N // E


class _Assign:
    def __init__(self, tl, el):
        self.token_labels, self.expert_labels = tl, el


class _Mat:
    def __init__(self, counts):
        self.counts = counts


@pytest.mark.parametrize("c", cases("simulate"), ids=["planted", "planted_noisy"])
def test_simulate_golden(c):
    rows = comm.simulate_trace(_Trace(c["tokens"], c["routed"]), _Topo(4, 16, 2),
                               _Assign(c["token_labels"], c["expert_labels"]),
                               _Mat(c["train_counts"]))
    assert [r["local_tokens"] for r in rows] == c["local"].tolist()
    assert [r["remote_tokens"] for r in rows] == c["remote"].tolist()
    assert np.array_equal([r["measured_alpha"] for r in rows], c["alpha"])
    assert np.allclose([r["pipeline_volume"] for r in rows], c["pipeline_volume"], rtol=0, atol=1e-9)
    assert np.allclose([r["saving"] for r in rows], c["saving"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("ci", range(3))
def test_toy_bundle_on_gpu(ci):
    """configs[0]: solver-built MDLB bundle -> HBM tables -> lookup / LAR."""
    c = cases("toy")[ci]
    b, dt = tables.load_device_tables(toy_bundle_path(ci))
    assert np.array_equal(S.lookup_devices(b, c["tokens"], c["hist"]), c["lookup_l2"])
    rows = comm.simulate_trace(_Trace(c["tokens"], c["routed"]), _Topo(2, 8, 2),
                               _Assign(c["token_labels"], c["expert_labels"]),
                               _Mat(c["train_counts"]))
    lar = []
    for mode in comm.MODES:
        loc = sum(r["local_tokens"] for r in rows if r["mode"] == mode)
        tot = sum(r["local_tokens"] + r["remote_tokens"] for r in rows if r["mode"] == mode)
        lar.append(loc / tot)
    assert np.array_equal(lar, c["lar"])
