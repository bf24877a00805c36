"""Generate the golden fixtures by running the REFERENCE (moesched) itself.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Only this script imports the reference; the committed .npz / .bin outputs
travel to the GPU box (where /root/reference does not exist) and pin both the
oracle (tests/test_oracle_golden.py) and the CUDA path (tests/test_gpu_golden.py).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from moesched import cli, comm, predictor, profiles, scheduler, solver, tables  # noqa: E402

OUT = Path(__file__).resolve().parent


def bundle_random(rng, E, vocab, n=2, zero_frac=0.3):
    labels = rng.integers(0, E, size=vocab)
    conf = rng.random(vocab).astype(np.float32)
    counts = rng.integers(0, 10, size=(E ** n, E))
    counts[rng.random(E ** n) < zero_frac] = 0
    tot = counts.sum(1, keepdims=True)
    probs = np.divide(counts, tot, out=np.zeros(counts.shape), where=tot > 0)
    tok = predictor.TokenDeviceTable(labels=labels, confidence=conf,
                                     provenance=np.zeros(vocab, np.uint8), n_clusters=E)
    ng = predictor.DeviceNGramTable(n=n, n_clusters=E, probs=probs, counts=counts)
    return scheduler.LookupBundle(token_table=tok, ngram_table=ng,
                                  expert_labels=np.arange(2 * E) % E, layers=4)


def lookup_cases():
    rng = np.random.default_rng(20261017)
    out = {}
    for ci, (E, vocab, n) in enumerate([(2, 16, 40), (4, 64, 300), (8, 1000, 5000),
                                        (16, 300, 2000)]):
        b = bundle_random(rng, E, vocab)
        tokens = rng.integers(-vocab, vocab, size=n)
        hist = rng.integers(0, E, size=(n, 2))
        out[f"c{ci}_labels"] = b.token_table.labels
        out[f"c{ci}_conf"] = b.token_table.confidence
        out[f"c{ci}_probs"] = b.ngram_table.probs
        out[f"c{ci}_counts"] = b.ngram_table.counts
        out[f"c{ci}_E"] = np.int64(E)
        out[f"c{ci}_tokens"] = tokens
        out[f"c{ci}_hist"] = hist
        out[f"c{ci}_dev_hist"] = scheduler.lookup_devices(b, tokens, hist)
        out[f"c{ci}_dev_static"] = scheduler.lookup_devices(b, tokens, None)
        # scalar twin on the first 20 tokens
        src = [scheduler.lookup_device(b, int(t), h) for t, h in zip(tokens[:20], hist[:20])]
        out[f"c{ci}_scalar_dev"] = np.array([s[0] for s in src])
        out[f"c{ci}_scalar_ngram"] = np.array([s[1] == "ngram" for s in src])
    out["n_cases"] = np.int64(4)
    np.savez_compressed(OUT / "lookup.npz", **out)


def rebatch_cases():
    rng = np.random.default_rng(7)
    out = {}
    cases = [(1, 2), (5, 2), (37, 3), (500, 4), (2049, 8), (4096, 8), (3000, 16), (100, 1)]
    for ci, (n, G) in enumerate(cases):
        tokens = rng.integers(0, 50_000, size=n)
        p = rng.dirichlet(np.ones(G) * 0.7)
        devices = rng.choice(G, size=n, p=p)
        sh, ix = scheduler.rebatch_tokens(tokens, devices, G)
        out[f"c{ci}_tokens"] = tokens
        out[f"c{ci}_devices"] = devices
        out[f"c{ci}_G"] = np.int64(G)
        out[f"c{ci}_shuffled"] = sh
        out[f"c{ci}_forward"] = ix.forward
        out[f"c{ci}_inverse"] = ix.inverse
        out[f"c{ci}_group"] = np.int64(ix.group_size)
        out[f"c{ci}_resumed"] = scheduler.resume_tokens(sh, ix)
    out["n_cases"] = np.int64(len(cases))
    np.savez_compressed(OUT / "rebatch.npz", **out)


def gate_cases():
    rng = np.random.default_rng(13)
    out = {}
    cases = [(4, 2), (16, 4), (64, 8), (8, 8), (60, 6)]
    for ci, (N, E) in enumerate(cases):
        labels = rng.permutation(np.arange(N) % E)
        perm = scheduler.gate_permutation(labels, E)
        logits = rng.normal(size=(9, N)).astype(np.float32)
        topk = rng.integers(0, N, size=(11, 3))
        out[f"c{ci}_labels"] = labels
        out[f"c{ci}_E"] = np.int64(E)
        out[f"c{ci}_new_to_old"] = perm.new_to_old
        out[f"c{ci}_old_to_new"] = perm.old_to_new
        out[f"c{ci}_logits"] = logits
        out[f"c{ci}_shuffled"] = scheduler.apply_expert_shuffle(logits, perm)
        out[f"c{ci}_topk"] = topk
        out[f"c{ci}_remapped"] = scheduler.remap_topk(topk, perm)
    out["n_cases"] = np.int64(len(cases))
    np.savez_compressed(OUT / "gate.npz", **out)


def aggregate(mats):
    total = np.zeros(mats[0].counts.shape, dtype=np.int64)
    for m in mats:
        total += m.counts.astype(np.int64)
    return profiles.TokenExpertMatrix(layer=-1, counts=total)


def simulate_cases():
    """comm.simulate_layer on the reference's own planted fixtures
    (tests/conftest.py:7-24) with the truth assignment (test_comm.py:91-117)."""
    out = {}
    for ci, (noise, seed) in enumerate([(0.0, 0), (0.2, 1)]):
        topo = profiles.Topology(devices=4, clusters=4, experts=16, top_k=2, layers=3,
                                 vocab=1024)
        mats, trace, truth = profiles.synthesize_planted_profile(
            topo, noise=noise, tokens_per_cluster=50, seed=seed, reps=8)
        tl = truth["token_labels"].copy()
        tl[tl < 0] = 0
        assign = solver.Assignment(token_labels=tl, expert_labels=truth["expert_labels"])
        agg = aggregate(mats)
        rows = comm.simulate_trace(trace, topo, assign, agg)
        out[f"c{ci}_tokens"] = trace.all_tokens()
        out[f"c{ci}_routed"] = trace.all_routed()
        out[f"c{ci}_token_labels"] = tl
        out[f"c{ci}_expert_labels"] = np.asarray(truth["expert_labels"])
        out[f"c{ci}_train_counts"] = agg.counts.astype(np.int64)
        out[f"c{ci}_local"] = np.array([r["local_tokens"] for r in rows])
        out[f"c{ci}_remote"] = np.array([r["remote_tokens"] for r in rows])
        out[f"c{ci}_alpha"] = np.array([r["measured_alpha"] for r in rows])
        out[f"c{ci}_mode"] = np.array([comm.MODES.index(r["mode"]) for r in rows])
        out[f"c{ci}_layer"] = np.array([r["layer"] for r in rows])
        out[f"c{ci}_pipeline_volume"] = np.array([r["pipeline_volume"] for r in rows])
        out[f"c{ci}_saving"] = np.array([r["saving"] for r in rows])
    out["n_cases"] = np.int64(2)
    np.savez_compressed(OUT / "simulate.npz", **out)


def toy_bundle():
    """configs[0] 'Reference CPU toy': G=E=2, N=8, k=2, L=3, planted 50
    tokens/cluster, solve_ceo(60 steps, 64 samples, eta 0.7, seed 0) +
    cli._build_bundle(n=2) -> MDLB bundle + the LAR of each mode."""
    out = {}
    for ci, noise in enumerate([0.0, 0.2, 0.5]):
        topo = profiles.Topology(devices=2, clusters=2, experts=8, top_k=2, layers=3, vocab=1024)
        mats, trace, truth = profiles.synthesize_planted_profile(
            topo, noise=noise, tokens_per_cluster=50, seed=0, reps=8)
        agg = aggregate(mats)
        cfg = solver.SolverConfig(theta=0.5, n_steps=60, n_samples=64, eta=0.7, seed=0)
        assign, _ = solver.solve_ceo(agg, cfg, topo)
        b = cli._build_bundle(topo, agg, trace, assign, 2)
        path = OUT / f"toy_eps{int(noise * 10)}.bin"
        tables.write_bundle(path, b)
        rows = comm.simulate_trace(trace, topo, assign, agg)
        lar = {}
        for mode in comm.MODES:
            loc = sum(r["local_tokens"] for r in rows if r["mode"] == mode)
            tot = sum(r["local_tokens"] + r["remote_tokens"] for r in rows if r["mode"] == mode)
            lar[mode] = loc / tot
        out[f"c{ci}_lar"] = np.array([lar[m] for m in comm.MODES])
        out[f"c{ci}_tokens"] = trace.all_tokens()
        out[f"c{ci}_routed"] = trace.all_routed()
        out[f"c{ci}_train_counts"] = agg.counts.astype(np.int64)
        out[f"c{ci}_token_labels"] = assign.token_labels
        out[f"c{ci}_expert_labels"] = assign.expert_labels
        # layer-2 lookup with the true previous-layer devices as histories
        routed = trace.all_routed()
        hist_dev = np.asarray(assign.expert_labels)[routed[:, :2, 0]]
        tokens = trace.all_tokens()
        out[f"c{ci}_hist"] = hist_dev
        out[f"c{ci}_lookup_l2"] = scheduler.lookup_devices(b, tokens, hist_dev)
        out[f"c{ci}_noise"] = np.float64(noise)
    out["n_cases"] = np.int64(3)
    np.savez_compressed(OUT / "toy.npz", **out)


def toy_chain():
    """configs[0] through the whole layer: the toy bundles of toy_bundle()
    driving a 3-layer chain.  Per layer the reference's own functions give the
    lookup (histories=None for the first n = 2 layers, scheduler.py:84-89;
    then the top-1 clusters of the previous two layers, predictor.py:157-166),
    the rebatch plan (rebatch_tokens) and -- through solver.metrics on a
    one-layer trace with those devices as token labels -- the local events."""
    out = {}
    toy = np.load(OUT / "toy.npz")
    for ci in range(3):
        b = tables.read_bundle(OUT / f"toy_eps{[0, 2, 5][ci]}.bin")
        tokens = toy[f"c{ci}_tokens"]
        routed = toy[f"c{ci}_routed"]
        C = np.asarray(b.expert_labels, dtype=np.int64)
        n = 2
        for layer in range(routed.shape[1]):
            hist = None if layer < n else C[routed[:, layer - n:layer, 0]]
            dev = scheduler.lookup_devices(b, tokens, hist)
            sh, ix = scheduler.rebatch_tokens(tokens, dev, 2)
            # metrics over this layer with the looked-up devices as the
            # "token labels" of each occurrence (occurrence i -> token id i)
            occ = np.arange(len(tokens))
            tr = profiles.RequestTrace(requests=((0, occ),), routed=(routed[:, layer:layer + 1],))
            m = solver.metrics(solver.Assignment(token_labels=dev, expert_labels=C), tr)
            pre = f"c{ci}_l{layer}_"
            out[pre + "dev"] = dev
            out[pre + "forward"] = ix.forward
            out[pre + "inverse"] = ix.inverse
            out[pre + "group"] = np.int64(ix.group_size)
            out[pre + "shuffled"] = sh
            out[pre + "local"] = np.int64(m["local_events"])
            out[pre + "imbalance"] = np.float64(m["imbalance"])
            if hist is not None:
                out[pre + "hist"] = hist
    out["n_cases"] = np.int64(3)
    np.savez_compressed(OUT / "toy_chain.npz", **out)


def metrics_cases():
    """solver.metrics (solver.py:766-800) on the reference's own planted
    fixtures (tests/conftest.py:7-24): truth assignment (test_solver.py:
    342-351: LAR 1.0, imbalance 1.0), a round-robin assignment and a solved
    one, each on the trace and on the aggregated count matrix."""
    out = {}
    ci = 0
    for noise, seed in ((0.0, 0), (0.2, 1)):
        topo = profiles.Topology(devices=4, clusters=4, experts=16, top_k=2, layers=3,
                                 vocab=1024)
        mats, trace, truth = profiles.synthesize_planted_profile(
            topo, noise=noise, tokens_per_cluster=50, seed=seed, reps=8)
        agg = aggregate(mats)
        R = truth["token_labels"].copy()
        R[R < 0] = 0
        assigns = [solver.Assignment(token_labels=R, expert_labels=truth["expert_labels"]),
                   solver.baseline_round_robin(topo)]
        cfg = solver.SolverConfig(n_steps=20, n_samples=32, eta=0.5, seed=seed)
        assigns.append(solver.solve_ceo(agg, cfg, topo)[0])
        for a in assigns:
            for kind, ev in (("trace", trace), ("matrix", agg)):
                m = solver.metrics(a, ev)
                pre = f"c{ci}_"
                out[pre + "kind"] = np.int64(kind == "trace")
                out[pre + "token_labels"] = np.asarray(a.token_labels, dtype=np.int64)
                out[pre + "expert_labels"] = np.asarray(a.expert_labels, dtype=np.int64)
                out[pre + "lar"] = np.float64(m["lar"])
                out[pre + "imbalance"] = np.float64(m["imbalance"])
                out[pre + "events"] = np.int64(m["events"])
                out[pre + "local_events"] = np.int64(m["local_events"])
                if kind == "trace":
                    out[pre + "tokens"] = trace.all_tokens()
                    out[pre + "routed"] = trace.all_routed()
                else:
                    out[pre + "counts"] = agg.counts.astype(np.int64)
                ci += 1
    out["n_cases"] = np.int64(ci)
    np.savez_compressed(OUT / "metrics.npz", **out)


def ceo_cases():
    """solve_ceo's per-iteration sample scoring (solver.py:380-404): samples
    drawn by the reference's own capacity-masked `sample_labels`, `joint`
    from the reference's `_sample_scores`, ep_scores / tk_scores with the
    expressions of solver.py:388-396 (the reference computes them inline)."""
    out = {}
    ci = 0
    specs = [(dict(devices=4, clusters=4, experts=16, top_k=2, layers=3, vocab=1024), 0.2, 32),
             (dict(devices=2, clusters=2, experts=8, top_k=2, layers=2, vocab=512), 0.5, 16),
             (dict(devices=8, clusters=8, experts=64, top_k=6, layers=2, vocab=4096), 0.3, 64)]
    for spec, noise, K in specs:
        topo = profiles.Topology(**spec)
        mats, trace, truth = profiles.synthesize_planted_profile(
            topo, noise=noise, tokens_per_cluster=40, seed=ci, reps=4)
        agg = aggregate(mats)
        active = np.nonzero(agg.freq > 0)[0]
        sub = profiles.TokenExpertMatrix(layer=agg.layer, counts=agg.counts[active])
        sub_counts = agg.counts[active].astype(np.float64)
        E, N = topo.clusters, topo.experts
        rng = np.random.default_rng(100 + ci)
        p_ep = rng.dirichlet(np.ones(E), size=N)
        p_tk = rng.dirichlet(np.ones(E), size=len(active))
        ep = solver.sample_labels(p_ep, "expert", None, 1.1, rng, K)
        tk = solver.sample_labels(p_tk, "token", sub, 1.1, rng, K)
        onehot = np.zeros((K, N, E))
        onehot[np.arange(K)[:, None], np.arange(N)[None, :], ep] = 1.0
        cm = np.tensordot(sub_counts, onehot, axes=([1], [1])).transpose(1, 0, 2)
        ep_scores = cm.max(axis=2).sum(axis=1)
        W = sub_counts @ p_ep
        tk_scores = W[np.arange(len(active))[None, :], tk].sum(axis=1)
        joint = solver._sample_scores(ep, tk, sub_counts)
        pre = f"c{ci}_"
        out[pre + "counts"] = agg.counts[active].astype(np.int64)
        out[pre + "ep"], out[pre + "tk"], out[pre + "p_ep"] = ep, tk, p_ep
        out[pre + "ep_scores"], out[pre + "tk_scores"], out[pre + "joint"] = ep_scores, tk_scores, joint
        ci += 1
    out["n_cases"] = np.int64(ci)
    np.savez_compressed(OUT / "ceo.npz", **out)


if __name__ == "__main__":
    lookup_cases()
    rebatch_cases()
    gate_cases()
    simulate_cases()
    toy_bundle()
    toy_chain()
    metrics_cases()
    ceo_cases()
    for p in sorted(OUT.glob("*.npz")) + sorted(OUT.glob("*.bin")):
        print(p.name, p.stat().st_size)
