"""Whole-layer parity: GPU SpecMoELayer vs the fp32 CPU oracle.

Bit-exact: plan (forward/inverse/group/counts), routing (ordered top-k
original expert ids), local/remote event counts, the SRS rows.
Tolerance: layer output, relative Frobenius error <= 1e-2 (north_star)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import layer_ref
from paper_2503_04398_b200 import SpecMoELayer, synth

TOL = 1e-2


def oracle_for(w):
    b = w.bundle
    return layer_ref.layer_forward(
        partials=w.partials, tokens=w.tokens, hist=w.hist, t_labels=b.token_table.labels,
        t_conf=b.token_table.confidence, a_best=b.ngram_table.best,
        a_conf=b.ngram_table.confidence, n_clusters=w.cfg["G"], expert_labels=w.expert_labels,
        gate_w=w.gate_w, w1=w.w1, w3=w.w3, w2=w.w2, k=w.cfg["k"])


CASES = [
    ("toy", 384, 0.2, {}),
    ("toy", 1, 0.0, {}),
    ("toy", 1000, 0.5, {"G": 8, "N": 16}),
    ("toy", 700, 0.3, {"G": 8, "N": 64, "k": 6, "d": 512, "f": 256}),
    ("toy", 500, 0.1, {"G": 4, "N": 64, "k": 8, "d": 256, "f": 384}),
    ("toy", 300, 0.1, {"G": 1, "N": 8, "k": 2}),
    ("toy", 512, 0.2, {"G": 8, "N": 8, "k": 1, "d": 4096, "f": 512}),
    ("toy", 333, 0.2, {"G": 4, "N": 24, "k": 3}),          # N' = 32 (tcgen05) / CUDA-core gate
    ("toy", 2000, 0.4, {"G": 8, "N": 32, "k": 4, "d": 1024, "f": 256}),
    ("toy", 4100, 0.2, {"G": 4, "N": 16, "k": 2, "d": 512, "f": 256}),   # whole-row movers (>= 2048 rows)
    # N' > 64 (tcgen05 gate only): DeepSeek-V2's 160 experts, 96 (N' = 128
    # with 32 masked slots), 256 experts over 16 shards
    ("toy", 900, 0.3, {"G": 8, "N": 160, "k": 6, "d": 512, "f": 256}),
    ("toy", 600, 0.2, {"G": 4, "N": 96, "k": 8, "d": 256, "f": 256}),
    ("toy", 300, 0.2, {"G": 16, "N": 256, "k": 8, "d": 256, "f": 256}),
]


@pytest.fixture(params=[1, 0], ids=["gate_tcgen05", "gate_mma_sync"])
def gate_kernel(request):
    """Run a test with each gate kernel: tcgen05 (default) and the mma.sync /
    CUDA-core kernels (SMOE_OPT_GATE_TENSOR = 0)."""
    from paper_2503_04398_b200 import _native as N
    lib = N.lib()
    old = lib.smoe_get_option(N.OPT_GATE_TENSOR)
    N.check(lib.smoe_set_option(N.OPT_GATE_TENSOR, request.param), "set_option")
    yield request.param
    N.check(lib.smoe_set_option(N.OPT_GATE_TENSOR, old), "set_option")


@pytest.mark.parametrize("name,n,eps,over", CASES)
def test_layer_matches_oracle(name, n, eps, over, gate_kernel):
    if over.get("N", 8) > 64 and gate_kernel == 0:
        pytest.skip("the mma.sync / CUDA-core gates cover N <= 64")
    w = synth.make_workload(name, n=n, eps=eps, seed=n, cfg_override=over)
    G = w.cfg["G"]
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"],
                         max_tokens=n + 7)
    out = layer.forward(torch.from_numpy(w.partials), w.tokens, w.hist).float().numpy()
    ref = oracle_for(w)
    ix = layer.plan_indices(n)
    assert ix.group_size == ref["group"]
    assert np.array_equal(ix.forward, ref["forward"])
    assert np.array_equal(ix.inverse, ref["inverse"])
    assert np.array_equal(layer.plan_counts.cpu().numpy(), ref["counts"])
    # SRS rows are bit-exact (fixed fp32 summation order, RNE to bf16)
    hs = layer.hs.float().cpu().numpy()
    for g in range(G):
        c = int(ref["counts"][g])
        assert np.array_equal(hs[g, :c], ref["h"][ref["forward"][g * ref["group"]:g * ref["group"] + c]])
    r = layer.routing(n)
    assert np.array_equal(r["experts"], ref["experts"])
    assert np.allclose(r["weights"], ref["weights"], rtol=1e-4, atol=1e-6)
    st = layer.stats()
    assert st["local_tokens"] == ref["local"] and st["remote_tokens"] == ref["remote"]
    # rows a per-destination-shard deduplicating dispatch would send
    owners = np.asarray(w.expert_labels)[ref["experts"]]
    want_rows = sum(len(set(owners[i].tolist()) - {int(ref["devices"][i])}) for i in range(n))
    assert st["remote_rows"] == want_rows
    err = np.linalg.norm(out - ref["out"]) / np.linalg.norm(ref["out"])
    assert err <= TOL, err
    # every shard's SAG copy is identical
    for g in range(G):
        assert torch.equal(layer.out[g, :n], layer.out[0, :n])


def test_layer_repeatable_and_graph_capturable():
    w = synth.make_workload("toy", n=256, eps=0.2, seed=5, cfg_override={"G": 4, "N": 16})
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=256)
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    layer.partial_views(256).copy_(torch.from_numpy(w.partials).to(torch.bfloat16))
    a = layer.run_device(tok, hist).clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        layer.run_device(tok, hist)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        layer.run_device(tok, hist)
    layer.out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(layer.out_view(256), a)


def _oracle(w, hist, **kw):
    b = w.bundle
    return layer_ref.layer_forward(
        partials=w.partials, tokens=w.tokens, hist=hist, t_labels=b.token_table.labels,
        t_conf=b.token_table.confidence, a_best=b.ngram_table.best,
        a_conf=b.ngram_table.confidence, n_clusters=w.cfg["G"], expert_labels=w.expert_labels,
        gate_w=w.gate_w, w1=w.w1, w3=w.w3, w2=w.w2, k=w.cfg["k"], **kw)


def test_layer_bias_no_renorm_no_history():
    w = synth.make_workload("toy", n=400, eps=0.2, seed=9, cfg_override={"G": 4, "N": 16})
    bias = np.random.default_rng(0).normal(scale=0.05, size=16).astype(np.float32)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=400,
                         gate_b=bias, renormalize=False)
    out = layer.forward(torch.from_numpy(w.partials), w.tokens, None).float().numpy()
    ref = _oracle(w, None, renorm=False, bias=bias)
    assert np.array_equal(layer.plan_indices(400).forward, ref["forward"])
    r = layer.routing(400)
    assert np.array_equal(r["experts"], ref["experts"])
    assert np.allclose(r["weights"], ref["weights"], rtol=1e-4, atol=1e-6)
    assert np.linalg.norm(out - ref["out"]) / np.linalg.norm(ref["out"]) <= TOL


def test_layer_empty_batch():
    w = synth.make_workload("toy", n=8, eps=0.2, seed=2)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=64)
    out = layer.forward(torch.zeros((2, 0, 256), dtype=torch.bfloat16), np.zeros(0, np.int64),
                        np.zeros((0, 2), np.int64))
    assert tuple(out.shape) == (0, 256)
    assert layer.stats()["local_tokens"] == 0


def test_layer_history_chain():
    """§8f rank 1: the n-gram window for the next layer is produced on the GPU
    (shift + cluster of the top-1 expert, predictor.py:165-166) and drives the
    next layer's lookup."""
    over = {"G": 4, "N": 16}
    w1 = synth.make_workload("toy", n=500, eps=0.3, seed=21, cfg_override=over)
    layer = SpecMoELayer(w1.bundle, w1.gate_w, w1.w1, w1.w3, w1.w2, top_k=2, max_tokens=500)
    layer.forward(torch.from_numpy(w1.partials), w1.tokens, w1.hist)
    ref1 = _oracle(w1, w1.hist)
    labels = np.asarray(w1.expert_labels)
    want = np.concatenate([w1.hist[:, 1:], labels[ref1["experts"][:, :1]]], axis=1)
    nh = layer.next_history(500).cpu().numpy()
    assert np.array_equal(nh, want)
    # layer 2 consumes it (same tables, new hidden states)
    w2 = synth.make_workload("toy", n=500, eps=0.3, seed=22, cfg_override=over)
    w2.bundle, w2.tokens = w1.bundle, w1.tokens
    out2 = layer.forward(torch.from_numpy(w2.partials), w2.tokens,
                         layer.next_history(500).clone())
    ref2 = layer_ref.layer_forward(
        partials=w2.partials, tokens=w2.tokens, hist=want, t_labels=w1.bundle.token_table.labels,
        t_conf=w1.bundle.token_table.confidence, a_best=w1.bundle.ngram_table.best,
        a_conf=w1.bundle.ngram_table.confidence, n_clusters=4, expert_labels=labels,
        gate_w=w1.gate_w, w1=w1.w1, w3=w1.w3, w2=w1.w2, k=2)
    assert np.array_equal(layer.plan_indices(500).forward, ref2["forward"])
    o = out2.float().numpy()
    assert np.linalg.norm(o - ref2["out"]) / np.linalg.norm(ref2["out"]) <= TOL


def test_forward_async_pipeline_matches_sync():
    """Pipelined serving API: double-buffered partials, H2D / compute / D2H on
    three streams; every batch must equal the synchronous forward."""
    over = {"G": 4, "N": 16}
    ws = [synth.make_workload("toy", n=n, eps=0.2, seed=30 + i, cfg_override=over)
          for i, n in enumerate((300, 257, 300, 12, 299))]
    base = ws[0]
    layer = SpecMoELayer(base.bundle, base.gate_w, base.w1, base.w3, base.w2, top_k=2,
                         max_tokens=300)
    want = []
    for w in ws:
        want.append(layer.forward(torch.from_numpy(w.partials).to(torch.bfloat16), w.tokens,
                                  w.hist).float().numpy())
    pins = [(torch.from_numpy(w.partials).to(torch.bfloat16).pin_memory(),
             torch.from_numpy(w.tokens).pin_memory(), torch.from_numpy(w.hist).pin_memory())
            for w in ws]
    outs = [torch.empty((300, 256), dtype=torch.bfloat16).pin_memory() for _ in range(len(ws))]
    handles = [layer.forward_async(p, t, h, out=outs[i][: len(t)]) for i, (p, t, h) in
               enumerate(pins)]
    for i, hd in enumerate(handles):
        got = hd.result().float().numpy()
        assert np.array_equal(got, want[i]), i
    # the synchronous path still works after pipelining (partial buffer rebound)
    again = layer.forward(torch.from_numpy(ws[1].partials).to(torch.bfloat16), ws[1].tokens,
                          ws[1].hist).float().numpy()
    assert np.array_equal(again, want[1])


def test_layer_errors_follow_the_reference():
    from paper_2503_04398_b200.scheduler import SchedulerError
    w = synth.make_workload("toy", n=200, eps=0.2, seed=4, cfg_override={"G": 4, "N": 16})
    parts = torch.from_numpy(w.partials).to(torch.bfloat16)
    # too many tokens for the buffers
    small = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=100)
    with pytest.raises(SchedulerError):
        small.forward(parts, w.tokens, w.hist)
    # wrong partial shape
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=200)
    with pytest.raises(SchedulerError):
        layer.forward(parts[:2], w.tokens, w.hist)
    # token id outside the vocabulary: numpy IndexError in the reference lookup
    bad = w.tokens.copy()
    bad[7] = 10 ** 6
    with pytest.raises(IndexError):
        layer.forward(parts, bad, w.hist)
    # expert-row capacity too small for the routed pairs
    tight = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=200,
                         expert_rows=16)
    with pytest.raises(SchedulerError):
        tight.forward(parts, w.tokens, w.hist)
    # the layer recovers after errors
    out = layer.forward(parts, w.tokens, w.hist)
    assert torch.isfinite(out.float()).all()


@pytest.mark.parametrize("n,M", [(600, 2), (601, 3), (100, 2)])
def test_microbatched_matches_single(n, M):
    """Micro-batched streams give bit-identical outputs and histories."""
    from paper_2503_04398_b200.layer import MicroBatchedSpecMoE
    over = {"G": 4, "N": 16}
    w = synth.make_workload("toy", n=n, eps=0.25, seed=40 + n, cfg_override=over)
    ref_layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=n)
    ref = ref_layer.forward(torch.from_numpy(w.partials).to(torch.bfloat16), w.tokens, w.hist)
    ref_hist = ref_layer.next_history(n).clone()
    mb = MicroBatchedSpecMoE(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=n,
                             microbatches=M)
    mb.partial_views(n).copy_(torch.from_numpy(w.partials).to(torch.bfloat16).cuda())
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    for _ in range(2):
        out = mb.run_device(tok, hist)
        torch.cuda.synchronize()
        mb.check_errors()
        assert torch.equal(out.cpu(), ref.cpu() if ref.is_cuda else ref)
        assert torch.equal(mb.next_history(n), ref_hist)
    st = mb.stats()
    rs = ref_layer.stats()
    assert st["local_tokens"] + st["remote_tokens"] == rs["local_tokens"] + rs["remote_tokens"]


def test_forward_async_error_surfaces_in_its_own_batch():
    """An out-of-vocabulary token in batch 1 raises in handle 1's result();
    batches 0 and 2 (queued around it) are unaffected."""
    over = {"G": 4, "N": 16}
    w = synth.make_workload("toy", n=200, eps=0.2, seed=8, cfg_override=over)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=200)
    parts = torch.from_numpy(w.partials).to(torch.bfloat16)
    want = layer.forward(parts, w.tokens, w.hist).float().numpy()
    bad = w.tokens.copy()
    bad[5] = 10 ** 6
    pp = parts.pin_memory()
    hh = torch.from_numpy(w.hist).pin_memory()
    toks = [torch.from_numpy(x).pin_memory() for x in (w.tokens, bad, w.tokens)]
    outs = [torch.empty((200, 256), dtype=torch.bfloat16).pin_memory() for _ in range(3)]
    hs = [layer.forward_async(pp, t, hh, out=outs[i]) for i, t in enumerate(toks)]
    assert np.array_equal(hs[0].result().float().numpy(), want)
    with pytest.raises(IndexError):
        hs[1].result()
    assert np.array_equal(hs[2].result().float().numpy(), want)


def test_graph_capture_replays_the_layer():
    """SpecMoELayer.capture: a CUDA-graph replay equals the eager forward,
    and picks up new partials / tokens written into the captured buffers."""
    over = {"G": 4, "N": 16}
    wa = synth.make_workload("toy", n=128, eps=0.2, seed=21, cfg_override=over)
    wb = synth.make_workload("toy", n=128, eps=0.2, seed=22, cfg_override=over)
    wb.bundle, wb.gate_w, wb.w1, wb.w3, wb.w2 = wa.bundle, wa.gate_w, wa.w1, wa.w3, wa.w2
    layer = SpecMoELayer(wa.bundle, wa.gate_w, wa.w1, wa.w3, wa.w2, top_k=2, max_tokens=128)
    want = [layer.forward(torch.from_numpy(w.partials).to(torch.bfloat16), w.tokens,
                          w.hist).clone() for w in (wa, wb)]
    tok = torch.as_tensor(wa.tokens, device="cuda")
    hist = torch.as_tensor(wa.hist, device="cuda")
    layer.partial_views(128).copy_(torch.from_numpy(wa.partials).to(torch.bfloat16))
    g = layer.capture(tok, hist)
    for w, ref in ((wb, want[1]), (wa, want[0])):
        layer.partial_views(128).copy_(torch.from_numpy(w.partials).to(torch.bfloat16))
        tok.copy_(torch.as_tensor(w.tokens))
        hist.copy_(torch.as_tensor(w.hist))
        g.replay()
        torch.cuda.synchronize()
        layer.check_errors()
        assert torch.equal(layer.out_view(128).cpu(), ref.cpu())


@pytest.mark.parametrize("over", [{"G": 8, "N": 64, "k": 6, "d": 2048, "f": 256},
                                  {"G": 8, "N": 64, "k": 8, "d": 3584, "f": 256},
                                  {"G": 8, "N": 8, "k": 2, "d": 4096, "f": 256},
                                  {"G": 4, "N": 40, "k": 5, "d": 512, "f": 256}])
def test_tcgen05_gate_matches_mma_gate(over):
    """Both gate kernels on the same layer: identical top-k ids and event
    counts, weights within fp32 accumulation-order noise (model-sized d)."""
    from paper_2503_04398_b200 import _native as N
    lib = N.lib()
    n = 3000
    w = synth.make_workload("toy", n=n, eps=0.3, seed=77, cfg_override=over)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=over["k"], max_tokens=n)
    parts = torch.from_numpy(w.partials).to(torch.bfloat16)
    res = {}
    try:
        for opt in (1, 0):
            N.check(lib.smoe_set_option(N.OPT_GATE_TENSOR, opt), "set_option")
            layer.forward(parts, w.tokens, w.hist)
            res[opt] = (layer.routing(n), layer.stats())
    finally:
        N.check(lib.smoe_set_option(N.OPT_GATE_TENSOR, 1), "set_option")
    (ra, sa), (rb, sb) = res[1], res[0]
    assert np.array_equal(ra["experts"], rb["experts"])
    assert np.allclose(ra["weights"], rb["weights"], rtol=1e-4, atol=1e-6)
    assert (sa["local_tokens"], sa["remote_tokens"]) == (sb["local_tokens"], sb["remote_tokens"])


def test_layer_all_tokens_on_one_shard_of_sixteen():
    """G = 16 shards, every token looked up to shard 3: fifteen empty groups
    (count 0), one full group; plan, routing, counts and output vs the oracle."""
    from paper_2503_04398_b200.predictor import TokenDeviceTable
    from paper_2503_04398_b200.scheduler import LookupBundle
    over = {"G": 16, "N": 64, "k": 4, "d": 256, "f": 256}
    n = 500
    w = synth.make_workload("toy", n=n, eps=0.3, seed=9, cfg_override=over)
    tt = w.bundle.token_table
    w.bundle = LookupBundle(
        token_table=TokenDeviceTable(labels=np.full_like(tt.labels, 3),
                                     confidence=np.full_like(tt.confidence, 2.0),
                                     provenance=tt.provenance, n_clusters=16),
        ngram_table=w.bundle.ngram_table, expert_labels=w.bundle.expert_labels, layers=1)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=4, max_tokens=n)
    out = layer.forward(torch.from_numpy(w.partials), w.tokens, w.hist).float().numpy()
    ref = oracle_for(w)
    counts = layer.plan_counts.cpu().numpy()
    assert counts[3] == n and counts.sum() == n
    assert np.array_equal(layer.plan_indices(n).forward, ref["forward"])
    assert np.array_equal(layer.routing(n)["experts"], ref["experts"])
    st = layer.stats()
    assert st["local_tokens"] == ref["local"] and st["remote_tokens"] == ref["remote"]
    assert np.linalg.norm(out - ref["out"]) / np.linalg.norm(ref["out"]) <= TOL


@pytest.mark.parametrize("over,renorm", [
    ({"G": 8, "N": 16, "k": 2, "d": 512, "f": 384}, True),
    ({"G": 8, "N": 64, "k": 6, "d": 512, "f": 256}, False),
    ({"G": 8, "N": 64, "k": 8, "d": 512, "f": 256}, True),
    ({"G": 4, "N": 40, "k": 4, "d": 512, "f": 256}, False)])
def test_batch_invariance_across_cuts(over, renorm):
    """A token's output (and routing, weights, next-layer history) is
    bit-identical whether it is processed in a 1100-token batch or in
    decode-sized pieces (1, 7, 64, 300, 728 tokens): no kernel's per-row
    arithmetic depends on the other rows of its batch, and the
    batch-size-dependent kernel choices (one-SM vs SM-pair GEMMs, row vs chunk
    movers, the gate's route fused at <= 128 tokens) are bit-identical; N = 64
    runs the gate's split (two threads per row) epilogue, N = 40 its N' = 48
    register tree."""
    n = 1100
    w = synth.make_workload("toy", n=n, eps=0.3, seed=99, cfg_override=over)
    parts = torch.from_numpy(w.partials).to(torch.bfloat16)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=over["k"], max_tokens=n,
                         renormalize=renorm)
    full = layer.forward(parts, w.tokens, w.hist).clone()
    full_hist = layer.next_history(n).clone()
    full_route = layer.routing(n)
    lo = 0
    for size in (1, 7, 64, 300, 728):
        hi = lo + size
        got = layer.forward(parts[:, lo:hi].contiguous(), w.tokens[lo:hi], w.hist[lo:hi])
        assert torch.equal(got, full[lo:hi]), (lo, hi)
        assert torch.equal(layer.next_history(size), full_hist[lo:hi])
        route = layer.routing(size)
        for key in route:
            assert np.array_equal(np.asarray(route[key]), np.asarray(full_route[key])[lo:hi]), key
        lo = hi
    assert lo == n


def test_microbatched_forward_api_single_process():
    """MicroBatchedSpecMoE.forward (host partials in, device output out) equals
    the plain layer, and its histories are the plain layer's."""
    from paper_2503_04398_b200.layer import MicroBatchedSpecMoE
    over = {"G": 4, "N": 16}
    n = 450
    w = synth.make_workload("toy", n=n, eps=0.25, seed=61, cfg_override=over)
    parts = torch.from_numpy(w.partials).to(torch.bfloat16)
    ref_layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=n)
    want = ref_layer.forward(parts, w.tokens, w.hist)
    mb = MicroBatchedSpecMoE(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=n,
                             microbatches=3)
    got = mb.forward(parts, w.tokens, w.hist)
    assert torch.equal(got.cpu(), want.cpu())
    assert torch.equal(mb.next_history(n), ref_layer.next_history(n))


@pytest.mark.parametrize("stages", [0x00, 0xff])
def test_programmatic_dependent_launch_is_bit_identical(stages):
    """Programmatic dependent launch changes only when kernels start: the
    layer with every stage launched early (0xff, including the up GEMM the
    default keeps on a plain launch) and with none (0x00, SMOE_OPT_PDL = 0),
    eager and graph-replayed, matches the default bit for bit."""
    from paper_2503_04398_b200 import _native as N
    lib = N.lib()
    over = {"G": 8, "N": 64, "k": 6, "d": 512, "f": 256}
    n = 900
    w = synth.make_workload("toy", n=n, eps=0.3, seed=17, cfg_override=over, device=True)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=6, max_tokens=n)
    layer.partial_views(n).copy_(w.partials)
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    layer.run_device(tok, hist)
    torch.cuda.synchronize()
    want, want_hist = layer.out_view(n).clone(), layer.next_history(n).clone()
    old = lib.smoe_get_option(N.OPT_PDL), lib.smoe_get_option(N.OPT_PDL_STAGES)
    try:
        N.check(lib.smoe_set_option(N.OPT_PDL, int(stages != 0)), "opt")
        N.check(lib.smoe_set_option(N.OPT_PDL_STAGES, stages), "opt")
        for _ in range(2):
            layer.out_view(n).zero_()
            layer.run_device(tok, hist)
            torch.cuda.synchronize()
            assert torch.equal(layer.out_view(n), want)
            assert torch.equal(layer.next_history(n), want_hist)
        g = layer.capture(tok, hist)
        layer.out_view(n).zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(layer.out_view(n), want)
    finally:
        N.check(lib.smoe_set_option(N.OPT_PDL, old[0]), "opt")
        N.check(lib.smoe_set_option(N.OPT_PDL_STAGES, old[1]), "opt")


@pytest.mark.parametrize("toggle", ["off_on", "on_off", "steady"])
def test_early_down_gemm_bit_identical(toggle):
    """SMOE_OPT_EARLY_DOWN (decode-sized batches: the down GEMM starts on the
    SMs the up GEMM's tail frees and waits per expert on counters the up
    GEMM's epilogue publishes) changes only when tiles start: outputs match
    the plain launch bit for bit, eager and graph-replayed -- also when the
    option flips between the EXPERT_UP and EXPERT_DOWN stage calls (the down
    GEMM only waits behind an up GEMM that published this forward's counts)."""
    from paper_2503_04398_b200 import _native as N
    lib = N.lib()
    over = {"G": 8, "N": 64, "k": 6, "d": 512, "f": 256}
    n = 64
    w = synth.make_workload("toy", n=n, eps=0.3, seed=23, cfg_override=over, device=True)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=6, max_tokens=n)
    layer.partial_views(n).copy_(w.partials)
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    old = lib.smoe_get_option(N.OPT_EARLY_DOWN)
    try:
        N.check(lib.smoe_set_option(N.OPT_EARLY_DOWN, 0), "opt")
        layer.run_device(tok, hist)
        torch.cuda.synchronize()
        layer.check_errors()
        want = layer.out_view(n).clone()
        up = list(range(N.STAGE_NAMES.index("expert_up") + 1))
        down = list(range(up[-1] + 1, len(N.STAGE_NAMES)))
        first, second = {"off_on": (0, 1), "on_off": (1, 0), "steady": (1, 1)}[toggle]
        for _ in range(2):
            layer.out_view(n).zero_()
            N.check(lib.smoe_set_option(N.OPT_EARLY_DOWN, first), "opt")
            layer.run_device(tok, hist, stages=up)
            N.check(lib.smoe_set_option(N.OPT_EARLY_DOWN, second), "opt")
            layer.run_device(tok, hist, stages=down)
            torch.cuda.synchronize()
            layer.check_errors()
            assert torch.equal(layer.out_view(n), want)
        N.check(lib.smoe_set_option(N.OPT_EARLY_DOWN, 1), "opt")
        g = layer.capture(tok, hist)
        layer.out_view(n).zero_()
        g.replay()
        torch.cuda.synchronize()
        layer.check_errors()
        assert torch.equal(layer.out_view(n), want)
    finally:
        N.check(lib.smoe_set_option(N.OPT_EARLY_DOWN, old), "opt")


@pytest.mark.parametrize("n,over", [(64, {"G": 8, "N": 64, "k": 6, "d": 512, "f": 256}),
                                    (100, {"G": 4, "N": 160, "k": 6, "d": 256, "f": 256}),
                                    (7, {"G": 16, "N": 16, "k": 2, "d": 256, "f": 256})])
def test_route_in_gate_bit_identical(n, over):
    """SMOE_OPT_ROUTE_IN_GATE (batches of <= 128 tokens: the gate ranks each
    shard's pairs and publishes its count row, the route kernel is skipped)
    gives the same outputs, pair counts and statistics as the route kernel --
    also with shards that receive no token (G = 16, 7 tokens)."""
    from paper_2503_04398_b200 import _native as N
    lib = N.lib()
    w = synth.make_workload("toy", n=n, eps=0.3, seed=29, cfg_override=over, device=True)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=over["k"], max_tokens=n)
    layer.partial_views(n).copy_(w.partials)
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    old = lib.smoe_get_option(N.OPT_ROUTE_IN_GATE)
    res = []
    try:
        for v in (0, 1):
            N.check(lib.smoe_set_option(N.OPT_ROUTE_IN_GATE, v), "opt")
            layer.counts_mat.fill_(-1)
            layer.run_device(tok, hist)
            torch.cuda.synchronize()
            layer.check_errors()
            st = layer.stats(n)
            res.append((layer.out_view(n).clone(), st["pair_counts"], st["local_tokens"],
                        st["remote_tokens"], layer.routing(n)["experts"]))
    finally:
        N.check(lib.smoe_set_option(N.OPT_ROUTE_IN_GATE, old), "opt")
    assert torch.equal(res[0][0], res[1][0])
    assert res[0][1] == res[1][1] and res[0][2:4] == res[1][2:4]
    assert np.array_equal(res[0][4], res[1][4])


def test_up_gemm_schedules_bit_identical_and_tuner():
    """The up GEMM's schedules (one SM per 128x256 tile; SM pair per 256x256
    tile with n-grouped order) give bit-identical layer outputs, and
    tune_gemm_order picks one of them and leaves it set (restored here)."""
    from paper_2503_04398_b200 import _native as N
    lib = N.lib()
    over = {"G": 4, "N": 8, "k": 2, "d": 512, "f": 256}
    n = 8192                                      # 2 048 rows per expert: past the one-SM range
    w = synth.make_workload("toy", n=n, eps=0.3, seed=31, cfg_override=over, device=True)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=n)
    layer.partial_views(n).copy_(w.partials)
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    old = (lib.smoe_get_option(N.OPT_GEMM_CTA_GROUP_UP), lib.smoe_get_option(N.OPT_GEMM_GROUP_M_UP))
    outs = []
    try:
        for cg, gm in ((1, 0), (2, -2), (2, 0), (1, -2)):
            N.check(lib.smoe_set_option(N.OPT_GEMM_CTA_GROUP_UP, cg), "opt")
            N.check(lib.smoe_set_option(N.OPT_GEMM_GROUP_M_UP, gm), "opt")
            layer.out_view(n).zero_()
            layer.run_device(tok, hist)
            torch.cuda.synchronize()
            layer.check_errors()
            outs.append(layer.out_view(n).clone())
        for o in outs[1:]:
            assert torch.equal(o, outs[0])
        res = layer.tune_gemm_order(tok, hist, rounds=2, reps=1)
        assert res["tuned"] and tuple(res["choice"]) in ((1, 0), (2, -2))
        assert (lib.smoe_get_option(N.OPT_GEMM_CTA_GROUP_UP),
                lib.smoe_get_option(N.OPT_GEMM_GROUP_M_UP)) == tuple(res["choice"])
        layer.run_device(tok, hist)
        torch.cuda.synchronize()
        assert torch.equal(layer.out_view(n), outs[0])
    finally:
        N.check(lib.smoe_set_option(N.OPT_GEMM_CTA_GROUP_UP, old[0]), "opt")
        N.check(lib.smoe_set_option(N.OPT_GEMM_GROUP_M_UP, old[1]), "opt")


def test_decode_path_errors_and_recovery():
    """At decode sizes (route fused into the gate, early-started down GEMM,
    plan-kernel resets) the reference's errors still surface -- capacity,
    token range -- and the next clean batch is right (the per-forward
    resets and readiness counters do not leak between batches)."""
    from paper_2503_04398_b200.scheduler import SchedulerError
    over = {"G": 8, "N": 64, "k": 6, "d": 512, "f": 256}
    n = 64
    w = synth.make_workload("toy", n=n, eps=0.3, seed=41, cfg_override=over)
    parts = torch.from_numpy(w.partials).to(torch.bfloat16)
    ref = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=6, max_tokens=n)
    want = ref.forward(parts, w.tokens, w.hist).clone()
    tight = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=6, max_tokens=n,
                         expert_rows=4)
    with pytest.raises(SchedulerError):
        tight.forward(parts, w.tokens, w.hist)
    bad = w.tokens.copy()
    bad[3] = 10 ** 7
    with pytest.raises(IndexError):
        ref.forward(parts, bad, w.hist)
    for _ in range(2):
        assert torch.equal(ref.forward(parts, w.tokens, w.hist), want)


@pytest.mark.parametrize("n,over", [(64, {"G": 8, "N": 64, "k": 6, "d": 512, "f": 256}),
                                    (3000, {"G": 4, "N": 8, "k": 2, "d": 512, "f": 256}),
                                    (300, {"G": 4, "N": 160, "k": 6, "d": 256, "f": 256})])
def test_expert_buffer_padding_never_reaches_outputs(n, over):
    """The expert-input / hidden buffers start as small noise (layer.py) and
    hold stale rows of earlier batches: rows past an expert's routed rows feed
    the padding of its GEMM tiles but must never reach an output.  Poisoning
    both buffers (and the gate and combine arenas) with NaN / inf leaves the
    layer's outputs and statistics bit-identical."""
    w = synth.make_workload("toy", n=n, eps=0.3, seed=43, cfg_override=over, device=True)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=over["k"], max_tokens=n)
    layer.partial_views(n).copy_(w.partials)
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    layer.run_device(tok, hist)
    torch.cuda.synchronize()
    layer.check_errors()
    want = layer.out_view(n).clone()
    st = layer.stats(n)
    want_stats = (st["pair_counts"], st["local_tokens"], st["remote_tokens"])
    assert torch.isfinite(want.float()).all()
    for poison in (float("nan"), float("inf")):
        # + the gate's input arena (rows past a shard's count fill the last
        # 128-row gate tile) and the combine's pair rows
        for buf in (layer.xin, layer.hmid, layer.hs, layer.ypair):
            buf.fill_(poison)
        layer.out_view(n).zero_()
        layer.run_device(tok, hist)
        torch.cuda.synchronize()
        layer.check_errors()
        assert torch.equal(layer.out_view(n), want)
        st = layer.stats(n)
        assert (st["pair_counts"], st["local_tokens"], st["remote_tokens"]) == want_stats


@pytest.mark.parametrize("up_pdl", [0, 1])
def test_decode_up_gemm_pdl_bit_identical(up_pdl):
    """SMOE_OPT_DECODE_UP_PDL: at decode sizes the up GEMM launches under PDL
    behind readiness counters the plan kernel resets (no memset node between
    the dispatch and the up GEMM).  Outputs equal the plain launch's bit for
    bit, eager, graph-replayed, and when an EXPERT_UP stage call runs twice
    without a PLAN in between (the counters are then reset by a memset)."""
    from paper_2503_04398_b200 import _native as N
    lib = N.lib()
    over = {"G": 8, "N": 64, "k": 6, "d": 512, "f": 256}
    n = 64
    w = synth.make_workload("toy", n=n, eps=0.3, seed=47, cfg_override=over, device=True)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=6, max_tokens=n)
    layer.partial_views(n).copy_(w.partials)
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    old = lib.smoe_get_option(N.OPT_DECODE_UP_PDL)
    try:
        N.check(lib.smoe_set_option(N.OPT_DECODE_UP_PDL, 0), "opt")
        layer.run_device(tok, hist)
        torch.cuda.synchronize()
        layer.check_errors()
        want = layer.out_view(n).clone()
        N.check(lib.smoe_set_option(N.OPT_DECODE_UP_PDL, up_pdl), "opt")
        for _ in range(3):
            layer.out_view(n).zero_()
            layer.run_device(tok, hist)
            torch.cuda.synchronize()
            layer.check_errors()
            assert torch.equal(layer.out_view(n), want)
        up = N.STAGE_NAMES.index("expert_up")
        layer.out_view(n).zero_()
        layer.run_device(tok, hist, stages=list(range(up + 1)))
        layer.run_device(tok, hist, stages=list(range(up, len(N.STAGE_NAMES))))
        torch.cuda.synchronize()
        layer.check_errors()
        assert torch.equal(layer.out_view(n), want)
        g = layer.capture(tok, hist)
        for _ in range(3):
            layer.out_view(n).zero_()
            g.replay()
            torch.cuda.synchronize()
            layer.check_errors()
            assert torch.equal(layer.out_view(n), want)
    finally:
        N.check(lib.smoe_set_option(N.OPT_DECODE_UP_PDL, old), "opt")
