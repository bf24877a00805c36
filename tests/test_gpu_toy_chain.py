"""configs[0] ("Reference CPU toy": 8 experts top-2, hidden 256, EP = 2
simulated ranks, solver-built E/T/S tables) through the whole GPU layer.

The MDLB bundles tests/golden/toy_eps{0,2,5}.bin were written by the
reference (solve_ceo + cli._build_bundle, make_golden.py).  A three-layer
chain runs `SpecMoELayer` on them with hidden states planted so the gate
reproduces the reference trace's routed experts; each layer's lookup, plan,
local events and imbalance are checked bit-exactly against the reference's own
functions (tests/golden/toy_chain.npz), the output against the fp32 oracle.
The history window follows the reference's contract: histories=None for the
first n = 2 layers (scheduler.py:84-89), then the top-1 clusters of the two
previous layers, produced on the GPU by the combine + SAG kernel.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from golden_util import cases, toy_bundle_path
from oracle import layer_ref
from paper_2503_04398_b200 import SpecMoELayer, metrics, synth, tables
from paper_2503_04398_b200.solver import Assignment, layer_metrics


@pytest.mark.parametrize("ci", range(3), ids=["eps0", "eps2", "eps5"])
def test_toy_bundle_layer_chain(ci):
    b = tables.read_bundle(toy_bundle_path(ci))
    toy, ch = cases("toy")[ci], cases("toy_chain")[ci]
    tokens, routed = toy["tokens"], toy["routed"]
    n, L, k = routed.shape
    d, f, G = 256, 512, 2
    C = np.asarray(b.expert_labels, dtype=np.int64)
    rng = np.random.default_rng(ci)
    gate = synth.planted_gate(8, d, rng)
    w1 = synth.bf16_round(rng.standard_normal((8, f, d)).astype(np.float32) / np.sqrt(d))
    w3 = synth.bf16_round(rng.standard_normal((8, f, d)).astype(np.float32) / np.sqrt(d))
    w2 = synth.bf16_round(rng.standard_normal((8, d, f)).astype(np.float32) / np.sqrt(f))
    layer = SpecMoELayer(b, gate, w1, w3, w2, top_k=k, max_tokens=n)
    assert layer.G == 2 and layer.history_width == 2
    win, depth = None, 0
    for l in range(L):
        partials = synth.planted_partials(gate, routed[:, l], G, rng)
        hist_in = None if win is None else win.clone()
        out = layer.forward(torch.from_numpy(partials), tokens, hist_in,
                            history_depth=depth if win is not None else None)
        pre = f"l{l}_"
        ix = layer.plan_indices(n)
        assert np.array_equal(layer.dev.cpu().numpy()[:n], ch[pre + "dev"])
        assert ix.group_size == int(ch[pre + "group"])
        assert np.array_equal(ix.forward, ch[pre + "forward"])
        assert np.array_equal(ix.inverse, ch[pre + "inverse"])
        r = layer.routing(n)
        assert np.array_equal(r["experts"], routed[:, l])
        st = layer.stats()
        assert st["local_tokens"] == int(ch[pre + "local"])
        assert st["local_tokens"] + st["remote_tokens"] == n * k
        m = layer_metrics(layer)
        assert m["imbalance"] == float(ch[pre + "imbalance"])
        ref = layer_ref.layer_forward(
            partials=partials, tokens=tokens,
            hist=None if hist_in is None else hist_in.cpu().numpy(), hist_depth=depth,
            t_labels=b.token_table.labels, t_conf=b.token_table.confidence,
            a_best=b.ngram_table.best, a_conf=b.ngram_table.confidence, n_clusters=2,
            expert_labels=C, gate_w=gate, w1=w1, w3=w3, w2=w2, k=k)
        got = out.float().numpy()
        assert np.linalg.norm(got - ref["out"]) / np.linalg.norm(ref["out"]) <= 1e-2
        win, depth = layer.history_window(n)
        assert depth == ref["next_depth"] == min(l + 1, 2)
        assert np.array_equal(win.cpu().numpy(), ref["next_window"])
        nh = layer.next_history(n)
        assert (nh is None) == (l == 0)
        if l + 1 < L and f"l{l + 1}_hist" in ch:
            assert np.array_equal(win.cpu().numpy(), ch[f"l{l + 1}_hist"])


class _Trace:
    def __init__(self, tokens, routed):
        self._t, self._r = tokens, routed

    def all_tokens(self):
        return self._t

    def all_routed(self):
        return self._r


class _Matrix:
    def __init__(self, counts):
        self.counts = counts


@pytest.mark.parametrize("c", cases("metrics"), ids=lambda c: "trace" if int(c["kind"]) else "matrix")
def test_metrics_on_gpu_match_reference(c):
    """solver.metrics (solver.py:766-800) through smoe_event_metrics vs the
    reference's values on its planted fixtures (test_solver.py:342-351)."""
    a = Assignment(token_labels=c["token_labels"], expert_labels=c["expert_labels"])
    ev = _Trace(c["tokens"], c["routed"]) if int(c["kind"]) else _Matrix(c["counts"])
    m = metrics(a, ev)
    assert m["lar"] == float(c["lar"]) and m["imbalance"] == float(c["imbalance"])
    assert m["events"] == int(c["events"]) and m["local_events"] == int(c["local_events"])


def test_history_inputs_validated_and_strided():
    """Strided token / history views give the same result as contiguous
    copies; a window of the wrong width is rejected (IndexError) instead of
    being read with the table's stride."""
    w = synth.make_workload("toy", n=300, eps=0.2, seed=12, cfg_override={"G": 4, "N": 16})
    parts = torch.from_numpy(w.partials).to(torch.bfloat16)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=300)
    want = layer.forward(parts, w.tokens, w.hist).clone()
    want_win = layer.next_history(300).clone()
    tok2 = torch.as_tensor(np.stack([w.tokens, w.tokens[::-1]], 1), device="cuda")[:, 0]
    wide = torch.as_tensor(np.concatenate([w.hist[:, :1] * 0 + 7, w.hist, w.hist], 1),
                           device="cuda")[:, 1:3]
    assert not tok2.is_contiguous() and not wide.is_contiguous()
    got = layer.forward(parts.cuda(), tok2, wide)
    assert torch.equal(got, want.cuda())
    assert torch.equal(layer.next_history(300), want_win)
    for bad in (w.hist[:, :1], np.concatenate([w.hist, w.hist[:, :1]], 1)):
        with pytest.raises(IndexError):
            layer.forward(parts, w.tokens, bad)
    # depth < width: T-only lookup (as histories=None), the window still shifts
    layer.forward(parts, w.tokens, w.hist, history_depth=1)
    none = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=300)
    none.forward(parts, w.tokens, None)
    assert np.array_equal(layer.plan_indices(300).forward, none.plan_indices(300).forward)
    win, depth = layer.history_window(300)
    assert depth == 2 and torch.equal(win[:, 0], torch.as_tensor(w.hist[:, 1], device="cuda"))
