"""fp32 CPU oracle of the whole speculative MoE layer (test oracle only).

The reference ships the index half (scheduler_ref) but none of the floating
point (SURVEY.md §8c "parity unpinned"); these functions follow the paper's
formulas and the layer contract in DESIGN.md:

  SRS      h[j] = bf16( sum_{r=0..G-1} P_r[forward[g*group + j]] )   fp32 adds in
           shard order r = 0..G-1 -> bit-exact target
  gate     logits = h . W_g^T (+ b);  top-k = first k of a stable argsort of
           -logits (lowest index on ties; test_scheduler.py:112 idiom);
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


def gate_topk(h: np.ndarray, gate_w: np.ndarray, k: int, renorm: bool, bias=None):
    logits = np.asarray(h, dtype=np.float64) @ np.asarray(gate_w, dtype=np.float64).T
    if bias is not None:
        logits = logits + np.asarray(bias, dtype=np.float64)
    order = np.argsort(-logits, axis=1, kind="stable")[:, :k]
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


def layer_forward(*, partials, tokens, hist, t_labels, t_conf, a_best, a_conf, n_clusters,
                  expert_labels, gate_w, w1, w3, w2, k, renorm=True, bias=None):
    """Whole-layer oracle.  Returns the layer output in the original order
    plus every intermediate the GPU path exposes."""
    G = int(n_clusters)
    dev = S.lookup_devices(t_labels, t_conf, a_best, a_conf, G, tokens, hist)
    forward, inverse, group, counts = S.rebatch_plan(dev, G)
    hs = srs(partials, forward, counts, group)
    n = len(tokens)
    d = np.asarray(partials).shape[2]
    h_orig = np.zeros((n, d), dtype=np.float32)        # reduced row of every token
    for g in range(G):
        h_orig[forward[g * group: g * group + int(counts[g])]] = hs[g]
    experts, weights, logits = gate_topk(h_orig, gate_w, k, renorm, bias)
    labels = np.asarray(expert_labels, dtype=np.int64)
    local = int(np.count_nonzero(labels[experts] == dev[:, None]))
    out = np.zeros((n, d), dtype=np.float32)
    for e in range(np.asarray(gate_w).shape[0]):
        rows, slots = np.nonzero(experts == e)
        if rows.size == 0:
            continue
        y = swiglu_expert(h_orig[rows], w1[e], w3[e], w2[e])
        out[rows] += weights[rows, slots][:, None] * y
    return {"out": out, "devices": dev, "forward": forward, "inverse": inverse,
            "group": group, "counts": counts, "h": h_orig, "experts": experts,
            "weights": weights, "logits": logits, "local": local,
            "remote": int(experts.size) - local}
