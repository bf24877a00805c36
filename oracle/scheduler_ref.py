"""numpy restatement of the reference's index arithmetic (test oracle only).

Every function cites the reference lines (under
/root/reference/pkg/src/moesched/) it restates.  Written independently of the
reference source: counting formulations instead of the reference's argsort
and Python loops, so agreement is a real cross-check.
"""

from __future__ import annotations

import numpy as np

PAD_TOKEN = -1


class OracleError(ValueError):
    pass


def history_rows(hist: np.ndarray, n_clusters: int) -> np.ndarray:
    """scheduler.py:91-93 / predictor.py:149-154: base-E code, oldest digit
    most significant (Horner evaluation in int64)."""
    hist = np.asarray(hist, dtype=np.int64)
    rows = np.zeros(hist.shape[0], dtype=np.int64)
    for j in range(hist.shape[1]):
        rows = rows * np.int64(n_clusters) + hist[:, j]
    return rows


def ngram_best_conf(probs: np.ndarray):
    """predictor.py:72-78: first argmax as int16, max as float32."""
    probs = np.asarray(probs, dtype=np.float64)
    return probs.argmax(axis=1).astype(np.int16), probs.max(axis=1).astype(np.float32)


def lookup_devices(t_labels, t_conf, a_best, a_conf, n_clusters, tokens, hist=None):
    """scheduler.py:82-98.  Strict float32 comparison; ties keep the token
    label; numpy wrap of negative ids (the reference indexes with them)."""
    tokens = np.asarray(tokens, dtype=np.int64)
    t_labels = np.asarray(t_labels, dtype=np.int16)
    t_conf = np.asarray(t_conf, dtype=np.float32)
    vocab = len(t_labels)
    if tokens.size and (tokens.min() < -vocab or tokens.max() >= vocab):
        raise IndexError("token id out of range")
    tok = np.where(tokens < 0, tokens + vocab, tokens)
    out = t_labels[tok].astype(np.int64)
    if hist is None:
        return out
    rows = history_rows(hist, n_clusters)
    R = len(a_conf)
    if rows.size and (rows.min() < -R or rows.max() >= R):
        raise IndexError("history row out of range")
    rows = np.where(rows < 0, rows + R, rows)
    a_conf = np.asarray(a_conf, dtype=np.float32)
    take = a_conf[rows] > t_conf[tok]
    out[take] = np.asarray(a_best, dtype=np.int64)[rows[take]]
    return out


def rebatch_plan(devices, n_devices: int):
    """scheduler.py:119-149, index half, as a counting sort:
    group = max per-device count; inverse[i] = d*group + (number of earlier
    tokens on d); forward is its inverse with -1 in the pads."""
    dev = np.asarray(devices, dtype=np.int64)
    if dev.size and (dev.min() < 0 or dev.max() >= n_devices):
        raise OracleError("device label out of range")
    counts = np.zeros(n_devices, dtype=np.int64)
    np.add.at(counts, dev, 1)
    group = int(counts.max()) if n_devices and dev.size else 0
    seen = np.zeros(n_devices, dtype=np.int64)
    inverse = np.empty(len(dev), dtype=np.int64)
    for i, d in enumerate(dev):            # stable by construction
        inverse[i] = d * group + seen[d]
        seen[d] += 1
    forward = np.full(n_devices * group, -1, dtype=np.int64)
    forward[inverse] = np.arange(len(dev), dtype=np.int64)
    return forward, inverse, group, counts


def rebatch_tokens(tokens, devices, n_devices: int):
    """scheduler.py:119-149 (ids): shuffled[s] = tokens[forward[s]] or PAD."""
    tokens = np.asarray(tokens)
    if len(tokens) != len(np.asarray(devices)):
        raise OracleError("tokens and devices must align")
    forward, inverse, group, _ = rebatch_plan(devices, n_devices)
    shuffled = np.full(len(forward), PAD_TOKEN, dtype=tokens.dtype)
    real = forward >= 0
    shuffled[real] = tokens[forward[real]]
    return shuffled, forward, inverse, group


def resume(shuffled, inverse):
    """scheduler.py:152-157."""
    return np.asarray(shuffled)[np.asarray(inverse, dtype=np.int64)]


def gate_permutation(labels, n_clusters: int):
    """scheduler.py:200-210: position of expert i = #experts with a smaller
    label + #earlier experts with the same label."""
    lab = np.asarray(labels, dtype=np.int64)
    if lab.size and (lab.min() < 0 or lab.max() >= n_clusters):
        raise OracleError("expert label out of range")
    N = len(lab)
    pos = np.array([np.sum(lab < lab[i]) + np.sum(lab[:i] == lab[i]) for i in range(N)],
                   dtype=np.int64)
    new_to_old = np.empty(N, dtype=np.int64)
    new_to_old[pos] = np.arange(N)
    return new_to_old, pos


def apply_expert_shuffle(logits, new_to_old):
    """scheduler.py:213-219."""
    return np.take(np.asarray(logits), np.asarray(new_to_old, dtype=np.int64), axis=-1)


def remap_topk(topk, old_to_new):
    """scheduler.py:222-224."""
    return np.asarray(old_to_new, dtype=np.int64)[np.asarray(topk, dtype=np.int64)]


def count_local(experts, expert_dev, token_dev) -> int:
    """comm.py:214: events whose expert sits on the token's device."""
    experts = np.asarray(experts, dtype=np.int64)
    ed = np.asarray(expert_dev, dtype=np.int64)[experts]
    return int(np.count_nonzero(ed == np.asarray(token_dev, dtype=np.int64)[:, None]))


def simulate_counts(tokens, routed_layer, mode, n_clusters, n_experts, token_labels=None,
                    expert_labels=None, train_counts=None):
    """comm.py:174-227 event counts for one layer under the three layouts."""
    occ = len(tokens)
    npc = n_experts // n_clusters
    if mode == "ds_moe":                     # comm.py:200-202
        expert_dev = np.arange(n_experts) // npc
        token_dev = np.arange(occ) % n_clusters
    elif mode == "s_ts":                     # comm.py:203-207, :160-168
        mass = np.asarray(train_counts, dtype=np.int64).reshape(
            len(train_counts), n_clusters, npc).sum(axis=2)
        expert_dev = np.arange(n_experts) // npc
        token_dev = mass.argmax(axis=1)[np.asarray(tokens)]
    else:                                    # comm.py:208-212
        expert_dev = np.asarray(expert_labels, dtype=np.int64)
        token_dev = np.asarray(token_labels, dtype=np.int64)[np.asarray(tokens)]
    local = count_local(routed_layer, expert_dev, token_dev)
    total = int(np.asarray(routed_layer).size)
    return local, total - local
