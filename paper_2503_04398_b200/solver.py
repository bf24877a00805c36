"""`moesched.solver` surface the online path needs: the assignment type and the
evaluation `metrics` (local activation rate + expert-side load imbalance,
reference solver.py:766-800), with the event counting on the GPU
(`smoe_event_metrics`).

The offline co-clustering search itself (`solve_ceo`, `solve_alternating`,
solver.py:200-760) is out of scope: it runs once per
deployment and is a sequential accept/reject search, not a data-parallel path.
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
