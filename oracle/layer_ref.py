"""fp32 CPU oracle of the whole speculative MoE layer (test oracle only).

The reference ships the index half (scheduler_ref) but none of the floating
point (SURVEY.md §8c "parity unpinned"); these functions follow the paper's
formulas and the layer contract in DESIGN.md:

  SRS      h[j] = bf16( sum_{r=0..G-1} P_r[forward[g*group + j]] )   fp32 adds in
           shard order r = 0..G-1 -> bit-exact target
  gate     logits = h . W_g^T (+ b);  top-k in s-EG SLOT space, the reference's
           own idiom (test_acceptance.py:179-193): shuffled =
           apply_expert_shuffle(logits) (scheduler.py:213-219), slots = first
           k of a stable argsort of -shuffled (lowest SLOT on exact ties;
           -inf logits are ordinary, lowest-slot-last candidates, so fewer
           than k finite logits still give k distinct experts), experts =
           new_to_old[slots] (remap, scheduler.py:222-224);
           weights = softmax(logits)[top-k], renormalised over the k when
           `renorm`
  expert   y = W2 . (silu(W1 . h) * (W3 . h))  (SwiGLU; external model fact)
  combine  out[i] = sum_s w_s * y_s ;  SAG places out at the original index
All inputs are bf16-valued float32 arrays; everything here is float64/float32.
"""

from __future__ import annotations

import numpy as np

from . import scheduler_ref as S


def bf16(x) -> np.ndarray:
    """Round float32 to the nearest bf16 (ties to even); returns float32."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    bits = a.view(np.uint32).astype(np.uint64)
    lsb = (bits >> np.uint64(16)) & np.uint64(1)
    rounded = ((bits + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
    return rounded.astype(np.uint32).view(np.float32).reshape(a.shape)


def srs(partials: np.ndarray, forward: np.ndarray, counts, group: int) -> list:
    """Per shard g: bf16 rows of token group g (real rows only)."""
    P = np.asarray(partials, dtype=np.float32)
    G = P.shape[0]
    out = []
    for g in range(G):
        src = forward[g * group: g * group + int(counts[g])]
        acc = P[0][src].copy()
        for r in range(1, G):
            acc = (acc + P[r][src]).astype(np.float32)
        out.append(bf16(acc))
    return out


def gate_topk(h: np.ndarray, gate_w: np.ndarray, k: int, renorm: bool, bias=None,
              new_to_old=None, logits=None):
    """Ordered top-k ORIGINAL expert ids, their weights and the logits.

    new_to_old: the s-EG slot order (gate_permutation, scheduler.py:200-210);
    ties are broken by slot, the reference's transparency idiom
    (test_acceptance.py:179-193).  None = identity (slot = expert id).
    logits: precomputed [n, N] logits (float64), e.g. to pin tie cases."""
    if logits is None:
        logits = np.asarray(h, dtype=np.float64) @ np.asarray(gate_w, dtype=np.float64).T
        if bias is not None:
            logits = logits + np.asarray(bias, dtype=np.float64)
    logits = np.asarray(logits, dtype=np.float64)
    N = logits.shape[1]
    n2o = np.arange(N) if new_to_old is None else np.asarray(new_to_old, dtype=np.int64)
    shuffled = S.apply_expert_shuffle(logits, n2o)
    slots = np.argsort(-shuffled, axis=1, kind="stable")[:, :k]
    order = n2o[slots]
    with np.errstate(invalid="ignore"):          # all -inf rows -> NaN weights, as on the GPU
        mx = logits.max(axis=1, keepdims=True)
        p = np.exp(logits - mx)
        p /= p.sum(axis=1, keepdims=True)
    w = np.take_along_axis(p, order, axis=1)
    if renorm:
        w = w / w.sum(axis=1, keepdims=True)
    return order.astype(np.int64), w.astype(np.float32), logits


def swiglu_expert(x: np.ndarray, w1: np.ndarray, w3: np.ndarray, w2: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float32)
    g = x @ np.asarray(w1, dtype=np.float32).T
    u = x @ np.asarray(w3, dtype=np.float32).T
    a = g / (1.0 + np.exp(-g)) * u
    return (a @ np.asarray(w2, dtype=np.float32).T).astype(np.float32)


def next_window(hist, hist_depth, top1_cluster, width):
    """The next layer's n-gram window (predictor.py:157-166: a history digit
    is the cluster of the top-1 routed expert, oldest digit first): drop the
    oldest digit, append this layer's top-1 cluster; digits not backed by an
    observed layer are 0 and the valid depth grows by one up to `width`
    (the reference passes histories=None for the first n layers,
    scheduler.py:84-89)."""
    n = len(top1_cluster)
    win = np.zeros((n, width), dtype=np.int64)
    if hist is not None and width > 1:
        win[:, :-1] = np.asarray(hist, dtype=np.int64)[:, 1:]
    win[:, -1] = np.asarray(top1_cluster, dtype=np.int64)
    depth = min((0 if hist is None else int(hist_depth)) + 1, width)
    win[:, : width - depth] = 0
    return win, depth


def layer_forward(*, partials, tokens, hist, t_labels, t_conf, a_best, a_conf, n_clusters,
                  expert_labels, gate_w, w1, w3, w2, k, renorm=True, bias=None,
                  hist_depth=None):
    """Whole-layer oracle.  Returns the layer output in the original order
    plus every intermediate the GPU path exposes.  `hist_depth` < the window
    width means the window is partial: the lookup is T-only, as for
    histories=None (scheduler.py:84-89)."""
    G = int(n_clusters)
    width = 0 if hist is None else np.asarray(hist).shape[1]
    depth = width if (hist is not None and hist_depth is None) else (hist_depth or 0)
    lookup_hist = hist if (hist is not None and depth >= width) else None
    dev = S.lookup_devices(t_labels, t_conf, a_best, a_conf, G, tokens, lookup_hist)
    forward, inverse, group, counts = S.rebatch_plan(dev, G)
    hs = srs(partials, forward, counts, group)
    n = len(tokens)
    d = np.asarray(partials).shape[2]
    h_orig = np.zeros((n, d), dtype=np.float32)        # reduced row of every token
    for g in range(G):
        h_orig[forward[g * group: g * group + int(counts[g])]] = hs[g]
    n2o, _ = S.gate_permutation(expert_labels, G)
    experts, weights, logits = gate_topk(h_orig, gate_w, k, renorm, bias, new_to_old=n2o)
    labels = np.asarray(expert_labels, dtype=np.int64)
    local = int(np.count_nonzero(labels[experts] == dev[:, None]))
    out = np.zeros((n, d), dtype=np.float32)
    for e in range(np.asarray(gate_w).shape[0]):
        rows, slots = np.nonzero(experts == e)
        if rows.size == 0:
            continue
        y = swiglu_expert(h_orig[rows], w1[e], w3[e], w2[e])
        out[rows] += weights[rows, slots][:, None] * y
    labels_top1 = labels[experts[:, 0]] if n else np.zeros(0, np.int64)
    win_w = width
    if hist is None:                       # the table depth: len(a_conf) == G ** n
        win_w = 0
        while G > 1 and G ** win_w < len(a_conf):
            win_w += 1
    window, wdepth = next_window(hist, depth, labels_top1, max(win_w, 1))
    return {"out": out, "devices": dev, "forward": forward, "inverse": inverse,
            "next_window": window, "next_depth": wdepth,
            "group": group, "counts": counts, "h": h_orig, "experts": experts,
            "weights": weights, "logits": logits, "local": local,
            "remote": int(experts.size) - local}


def metrics(token_labels, expert_labels, *, counts=None, tokens=None, routed=None):
    """solver.py:766-800 restated: LAR over activation events and the
    expert-side load imbalance max / median per cluster.  Either a count
    matrix (events weighted by counts) or a routed trace (tokens [occ],
    routed [occ, L, k], one event per entry)."""
    C = np.asarray(expert_labels, dtype=np.int64)
    R = np.asarray(token_labels, dtype=np.int64)
    E = int(C.max(initial=0)) + 1
    if counts is not None:
        counts = np.asarray(counts, dtype=np.int64)
        total = int(counts.sum())
        same = C[None, :] == R[: counts.shape[0]][:, None]
        local = int(counts[same].sum())
        loads = np.array([counts[:, C == c].sum() for c in range(E)], dtype=np.float64)
    else:
        routed = np.asarray(routed, dtype=np.int64)
        dev = R[np.asarray(tokens, dtype=np.int64)]
        ed = C[routed]
        local = int(np.count_nonzero(ed == dev[:, None, None]))
        total = int(ed.size)
        loads = np.bincount(ed.reshape(-1), minlength=E).astype(np.float64)
    med = float(np.median(loads))
    return {"lar": local / total, "imbalance": float(loads.max() / med) if med > 0 else np.inf,
            "events": total, "local_events": local}
