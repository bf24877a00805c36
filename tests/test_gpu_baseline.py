"""DS-MoE baseline pipeline (AR -> A2A -> A2A -> AG) vs the fp32 oracle, and
its event counts vs the reference's ds_moe layout (comm.py:200-202)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import layer_ref, scheduler_ref as R
from paper_2503_04398_b200 import synth
from paper_2503_04398_b200.baseline import DSMoELayer


@pytest.mark.parametrize("n,over", [(300, {"G": 2, "N": 8}), (1000, {"G": 8, "N": 16}),
                                    (777, {"G": 8, "N": 64, "k": 6, "d": 512, "f": 256})])
def test_dsmoe_matches_oracle(n, over):
    w = synth.make_workload("toy", n=n, eps=0.3, seed=n, cfg_override=over)
    G, k = w.cfg["G"], w.cfg["k"]
    b = w.bundle
    ref = layer_ref.layer_forward(partials=w.partials, tokens=w.tokens, hist=w.hist,
                                  t_labels=b.token_table.labels, t_conf=b.token_table.confidence,
                                  a_best=b.ngram_table.best, a_conf=b.ngram_table.confidence,
                                  n_clusters=G, expert_labels=w.expert_labels, gate_w=w.gate_w,
                                  w1=w.w1, w3=w.w3, w2=w.w2, k=k)
    layer = DSMoELayer(w.gate_w, w.w1, w.w3, w.w2, n_ranks=G, top_k=k, max_tokens=n)
    parts = [torch.from_numpy(w.partials[g]).cuda().to(torch.bfloat16) for g in range(G)]
    out = layer.forward(parts, n).float().cpu().numpy()
    err = np.linalg.norm(out - ref["out"]) / np.linalg.norm(ref["out"])
    assert err <= 1e-2, err
    st = layer.stats()
    loc, rem = R.simulate_counts(w.tokens, ref["experts"], "ds_moe", G, w.cfg["N"])
    assert (st["local_tokens"], st["remote_tokens"]) == (loc, rem)
    # the per-expert routed counts equal the oracle's expert histogram
    C = layer.last["counts"]
    assert np.array_equal(C.sum(0), np.bincount(ref["experts"].ravel(), minlength=w.cfg["N"]))


def _run_dsmoe_procs(world, over, n, backend):
    import socket
    import torch.multiprocessing as mp
    import mp_worker
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=mp_worker.dsmoe_worker, args=(r, world, port, over, n, backend, q))
             for r in range(world)]
    for p in procs:
        p.start()
    return mp_worker.collect(q, procs)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,over", [(2, {"G": 2, "N": 8}), (4, {"G": 4, "N": 16})])
def test_dsmoe_distributed_path(world, over):
    """DSMoELayer(distributed=True), the collective branch of comm.py:99-108
    (all_reduce -> all_to_all_single x2 -> all_gather_into_tensor): with one
    GPU per rank over NCCL (<= 1e-2 of the emulation: NCCL sums bf16 in ring
    order), else ranks sharing the GPU over gloo with host-staged collectives
    (bit-identical to the single-process emulation)."""
    n = 500
    nccl = torch.cuda.device_count() >= world
    res = _run_dsmoe_procs(world, over, n, "nccl" if nccl else "gloo")
    w = synth.make_workload("toy", n=n, eps=0.3, seed=5, cfg_override=over)
    ref_layer = DSMoELayer(w.gate_w, w.w1, w.w3, w.w2, n_ranks=world, top_k=w.cfg["k"],
                           max_tokens=n)
    parts = [torch.from_numpy(w.partials[g]).cuda().to(torch.bfloat16) for g in range(world)]
    ref = ref_layer.forward(parts, n).float().cpu().numpy()
    st = ref_layer.stats()
    loc = rem = 0
    for r in range(world):
        outs, (l, m) = res[r]
        loc, rem = loc + l, rem + m
        for o in outs:
            if nccl:
                assert np.linalg.norm(o - ref) / np.linalg.norm(ref) <= 1e-2
            else:
                assert np.array_equal(o, ref)
    # every rank counts its own tokens' pairs: the sum is the emulation's
    assert (loc, rem) == (st["local_tokens"], st["remote_tokens"])


# ---------------------------------------------------------------- like-for-like pipeline
from paper_2503_04398_b200.baseline import DSMoEPipelineLayer, position_bundle  # noqa: E402


def _dsmoe_oracle(w, n, partials=None):
    """The DS-MoE pipeline's math is the layer's with position sharding and
    contiguous experts: the same oracle, run on the position bundle."""
    G, N, k = w.cfg["G"], w.cfg["N"], w.cfg["k"]
    pb = position_bundle(n, G, N)
    return layer_ref.layer_forward(
        partials=w.partials if partials is None else partials, tokens=np.arange(n), hist=None,
        t_labels=pb.token_table.labels, t_conf=pb.token_table.confidence,
        a_best=pb.ngram_table.best, a_conf=pb.ngram_table.confidence, n_clusters=G,
        expert_labels=np.asarray(pb.expert_labels, dtype=np.int64), gate_w=w.gate_w,
        w1=w.w1, w3=w.w3, w2=w.w2, k=k)


@pytest.mark.parametrize("n,over", [(300, {"G": 2, "N": 8}), (1000, {"G": 8, "N": 16}),
                                    (777, {"G": 8, "N": 64, "k": 6, "d": 512, "f": 256}),
                                    (2600, {"G": 4, "N": 8}),
                                    # decode sizes: route fused into the gate, early down GEMM
                                    (64, {"G": 8, "N": 64, "k": 6, "d": 512, "f": 256}),
                                    (100, {"G": 4, "N": 8})])
def test_dsmoe_pipeline_matches_oracle(n, over):
    """SMOE_PIPELINE_DSMOE (all-reduce + slice, combine into all-gather blocks
    + resume) on the s-MoE kernels: plan = position sharding (comm.py:202),
    routing bit-exact, event counts = the reference's ds_moe layout
    (comm.py:200-202), output within the north-star tolerance; and the same
    result as the collective DSMoELayer emulation."""
    w = synth.make_workload("toy", n=n, eps=0.3, seed=n, cfg_override=over)
    G, k = w.cfg["G"], w.cfg["k"]
    ref = _dsmoe_oracle(w, n)
    layer = DSMoEPipelineLayer(w.gate_w, w.w1, w.w3, w.w2, n_ranks=G, top_k=k, max_tokens=n)
    out = layer.forward(torch.from_numpy(w.partials)).float().cpu().numpy()
    ix = layer.plan_indices(n)
    assert np.array_equal(layer.dev.cpu().numpy()[:n], np.arange(n) % G)
    assert np.array_equal(ix.forward, ref["forward"])
    r = layer.routing(n)
    assert np.array_equal(r["experts"], ref["experts"])
    st = layer.stats()
    loc, rem = R.simulate_counts(np.arange(n), ref["experts"], "ds_moe", G, w.cfg["N"])
    assert (st["local_tokens"], st["remote_tokens"]) == (loc, rem)
    err = np.linalg.norm(out - ref["out"]) / np.linalg.norm(ref["out"])
    assert err <= 1e-2, err
    # every rank received the full all-reduce (natural order, fp32 sum in rank order)
    ar = layer.ar_local[:n].float().cpu().numpy()
    assert np.array_equal(ar, ref["h"])
    coll = DSMoELayer(w.gate_w, w.w1, w.w3, w.w2, n_ranks=G, top_k=k, max_tokens=n)
    parts = [torch.from_numpy(w.partials[g]).cuda().to(torch.bfloat16) for g in range(G)]
    o2 = coll.forward(parts, n).float().cpu().numpy()
    assert np.linalg.norm(out - o2) / np.linalg.norm(o2) <= 1e-2


def test_dsmoe_pipeline_capacity_and_replay():
    """Batches smaller than the capacity, and CUDA-graph capture of the whole
    DS-MoE pipeline, give the plain forward's output bit for bit."""
    over = {"G": 8, "N": 16}
    w = synth.make_workload("toy", n=900, eps=0.3, seed=3, cfg_override=over)
    layer = DSMoEPipelineLayer(w.gate_w, w.w1, w.w3, w.w2, n_ranks=8, top_k=2, max_tokens=1024)
    parts = torch.from_numpy(w.partials).cuda()
    want = layer.forward(parts).clone()
    for n in (1, 7, 64, 900):
        o = layer.forward(parts[:, :n]).float().cpu().numpy()
        ref = _dsmoe_oracle(w, n, w.partials[:, :n])
        assert np.linalg.norm(o - ref["out"]) <= 1e-2 * np.linalg.norm(ref["out"])
    g = layer.capture(layer.positions(900))
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(layer.out_view(900), want)
    assert torch.equal(layer.forward(parts), want)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,over", [(2, {"G": 2, "N": 8}), (4, {"G": 8, "N": 16})])
def test_dsmoe_pipeline_multiprocess(world, over):
    """The like-for-like DS-MoE pipeline over a ShardGroup (CUDA IPC peer
    stores, one GPU per process when the box has them) is bit-identical to
    the single-process run."""
    import socket
    import torch.multiprocessing as mp
    import mp_worker
    n = 600
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=mp_worker.dsmoe_pipeline_worker, args=(r, world, port, over, n, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = mp_worker.collect(q, procs)
    w = synth.make_workload("toy", n=n, eps=0.3, seed=12, cfg_override=over)
    layer = DSMoEPipelineLayer(w.gate_w, w.w1, w.w3, w.w2, n_ranks=w.cfg["G"], top_k=w.cfg["k"],
                               max_tokens=n)
    want = layer.forward(torch.from_numpy(w.partials).cuda()).float().cpu().numpy()
    st = layer.stats_t.cpu().numpy()[:2]
    loc = rem = 0
    for r in range(world):
        outs, (l, m) = res[r]
        loc, rem = loc + l, rem + m
        for o in outs:
            assert np.array_equal(o, want)
    assert (loc, rem) == (int(st[0]), int(st[1]))
