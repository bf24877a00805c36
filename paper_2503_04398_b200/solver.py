"""`moesched.solver` surface the online path needs: the assignment type and the
evaluation `metrics` (local activation rate + expert-side load imbalance,
reference solver.py:766-800), with the event counting on the GPU
(`smoe_event_metrics`).

The offline co-clustering search itself (`solve_ceo`, `solve_alternating`,
solver.py:200-760) runs once per deployment; its sequential greedy polish
stays on the host.  Its one batched dense step -- scoring the
K sampled (expert, token) labelings of every cross-entropy iteration
(solver.py:380-404) -- runs on the GPU: `ceo_sample_scores`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _dev, _native


class SolverError(ValueError):
    pass


@dataclass
class Assignment:
    """Cluster of every token (R) and of every expert (C), solver.py:40-46."""

    token_labels: np.ndarray
    expert_labels: np.ndarray


def _event_metrics(experts, weights, occ, k, expert_dev, token_dev, n_clusters):
    """(local, loads[n_clusters]) over occ x k events, counted on the GPU."""
    L = _native.lib()
    t = _dev.torch()
    ed = _dev.to_device(np.asarray(expert_dev, dtype=np.int64))
    td = _dev.to_device(np.asarray(token_dev, dtype=np.int64))
    ex = None if experts is None else _dev.to_device(np.asarray(experts, dtype=np.int64))
    wt = None if weights is None else _dev.to_device(np.asarray(weights, dtype=np.int64))
    local = t.zeros(1, dtype=t.int64, device=ed.device)
    loads = t.zeros(n_clusters, dtype=t.int64, device=ed.device)
    err = _dev.ErrFlag()
    _native.check(L.smoe_event_metrics(_native.ptr(ex), _native.ptr(wt), int(occ), int(k),
                                       _native.ptr(ed), int(ed.numel()), _native.ptr(td),
                                       int(n_clusters), _native.ptr(local), _native.ptr(loads),
                                       err.ptr, _native.stream_ptr()), "event_metrics")
    if err.bits():
        raise IndexError("an expert id is outside the expert labels")
    return int(local.item()), loads.cpu().numpy()


def metrics(assign, evaluation) -> dict:
    """Local activation rate and load imbalance under an assignment
    (solver.py:766-800).

    evaluation: a token x expert count matrix (anything with `.counts`,
    counts-weighted events) or a routed trace (anything with `all_routed()` /
    `all_tokens()`, one event per (occurrence, layer, k-slot)).  LAR = local
    events / events; imbalance = max / median of the per-cluster expert-side
    load (inf when the median is 0)."""
    C = np.asarray(assign.expert_labels, dtype=np.int64)
    R = np.asarray(assign.token_labels, dtype=np.int64)
    E = int(C.max(initial=0)) + 1
    if hasattr(evaluation, "counts") and not hasattr(evaluation, "all_routed"):
        counts = np.asarray(evaluation.counts, dtype=np.int64)
        total = int(counts.sum())
        if total == 0:
            raise SolverError("no activation events to evaluate")
        T, N = counts.shape
        tok_dev = R[:T]
        if len(tok_dev) < T:                    # numpy: R[:T] shorter -> broadcast error
            raise ValueError("token labels do not cover the count matrix")
        local, loads = _event_metrics(None, counts, T, N, C[:N], tok_dev, E)
    elif hasattr(evaluation, "all_routed"):
        routed = np.asarray(evaluation.all_routed(), dtype=np.int64)
        tokens = np.asarray(evaluation.all_tokens(), dtype=np.int64)
        if routed.size == 0:
            raise SolverError("no activation events to evaluate")
        dev = R[tokens]                          # numpy semantics (IndexError / wrap)
        per_occ = int(np.prod(routed.shape[1:]))
        local, loads = _event_metrics(routed.reshape(len(tokens), per_occ), None, len(tokens),
                                      per_occ, C, dev, E)
        total = int(routed.size)
    else:
        raise SolverError("unsupported evaluation payload")
    loads = loads.astype(np.float64)
    median = float(np.median(loads))
    imbalance = float(loads.max() / median) if median > 0 else math.inf
    return {"lar": local / total, "imbalance": imbalance, "events": total,
            "local_events": int(local)}


def layer_metrics(layer) -> dict:
    """The same metrics for the last forward of a `SpecMoELayer`, from the
    [G, N] pair-count matrix its route stage publishes (no extra kernel):
    LAR = measured alpha, loads[c] = pairs routed to experts of cluster c."""
    st = layer.stats()
    cm = np.asarray(st["pair_counts"], dtype=np.int64)       # [G, N] in s-EG slot order
    owner = np.asarray(layer.slot_owner, dtype=np.int64)
    loads = np.bincount(owner, weights=cm.sum(axis=0), minlength=layer.G).astype(np.float64)
    total = st["local_tokens"] + st["remote_tokens"]
    median = float(np.median(loads))
    return {"lar": st["local_tokens"] / total if total else 0.0,
            "imbalance": float(loads.max() / median) if median > 0 else math.inf,
            "events": total, "local_events": st["local_tokens"], "loads": loads.tolist()}


def ceo_sample_scores(counts, ep_samples, tk_samples, p_ep=None):
    """One iteration's sample scores of solve_ceo (solver.py:380-404).

    counts: [t, N] activation counts of the active tokens (the reference's
    `sub_counts`); ep_samples int [K, N] and tk_samples int [K, t] cluster
    labels.  Returns (ep_scores, tk_scores, joint), float64 [K] each:

      ep_scores[k] = sum_j max_c cluster_mass[k, j, c]        (:388-393)
      joint[k]     = sum_j cluster_mass[k, j, tk[k, j]]       (:397-399)
      tk_scores[k] = sum_j (counts @ p_ep)[j, tk[k, j]]       (:395-396)

    ep_scores and joint (the K x t x N tensordot) come from the GPU as exact
    integer sums, so they equal the reference's float64 values bit for bit;
    tk_scores (a float64 reduction the reference does with numpy's pairwise
    sum) is only computed when p_ep is given, on the host with the reference's
    own expression so it too is bit-identical.
    """
    L = _native.lib()
    t = _dev.torch()
    c = np.asarray(counts)
    if c.ndim != 2:
        raise SolverError("counts must be [tokens, experts]")
    ep = np.asarray(ep_samples, dtype=np.int64)
    tk = np.asarray(tk_samples, dtype=np.int64)
    T, N = c.shape
    K = ep.shape[0]
    if ep.shape != (K, N) or tk.shape != (K, T):
        raise SolverError("sample shapes do not match the count matrix")
    E = int(max(ep.max(initial=0), tk.max(initial=0))) + 1
    if ep.size and ep.min() < 0 or tk.size and tk.min() < 0:
        raise SolverError("cluster labels must be non-negative")
    if c.size and (c.min() < 0 or c.max() > np.iinfo(np.int32).max):
        raise SolverError("counts must be non-negative int32 values")
    cnt = _dev.to_device(np.ascontiguousarray(c.T, dtype=np.int32))
    ep_d = _dev.to_device(np.ascontiguousarray(ep, dtype=np.int32))
    tk_d = _dev.to_device(np.ascontiguousarray(tk, dtype=np.int32))
    es = t.empty(max(K, 1), dtype=t.int64, device=cnt.device)
    js = t.empty(max(K, 1), dtype=t.int64, device=cnt.device)
    _native.check(L.smoe_ceo_sample_scores(_native.ptr(cnt), T, N, _native.ptr(ep_d),
                                           _native.ptr(tk_d), K, E, _native.ptr(es),
                                           _native.ptr(js), _native.stream_ptr()),
                  "ceo_sample_scores")
    ep_scores = es[:K].cpu().numpy().astype(np.float64)
    joint = js[:K].cpu().numpy().astype(np.float64)
    tk_scores = None
    if p_ep is not None:
        W = np.asarray(c, dtype=np.float64) @ np.asarray(p_ep, dtype=np.float64)
        tk_scores = W[np.arange(T)[None, :], tk].sum(axis=1)
    return ep_scores, tk_scores, joint
