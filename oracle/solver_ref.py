"""numpy restatement of solve_ceo's sample scoring (test oracle only).

Reference: /root/reference/pkg/src/moesched/solver.py:380-404 (inside
solve_ceo).  The reference builds a [K, N, E] one-hot, tensordots it with the
[t, N] counts into a [K, t, E] float64 tensor and reduces it; restated here
per sample with a cluster-by-expert indicator product and integer sums, so
agreement with the reference's float64 is a real cross-check (pinned by
tests/golden/ceo.npz, made by running the reference).
"""

from __future__ import annotations

import numpy as np


def ceo_scores(counts, ep_samples, tk_samples, p_ep=None):
    """(ep_scores, tk_scores | None, joint) as float64 [K]:
    ep_scores[k] = sum_j max_c mass[k, j, c] (solver.py:388-393),
    joint[k] = sum_j mass[k, j, tk[k, j]] (:397-399),
    tk_scores[k] = sum_j (counts @ p_ep)[j, tk[k, j]] (:395-396),
    mass[k, j, c] = sum of counts[j, n] over experts n labelled c in ep[k]."""
    c = np.asarray(counts, dtype=np.int64)
    ep = np.asarray(ep_samples, dtype=np.int64)
    tk = np.asarray(tk_samples, dtype=np.int64)
    T = c.shape[0]
    E = int(max(ep.max(initial=0), tk.max(initial=0))) + 1
    ep_scores = np.zeros(len(ep))
    joint = np.zeros(len(ep))
    for k in range(len(ep)):
        ind = np.zeros((c.shape[1], E), dtype=np.int64)
        ind[np.arange(c.shape[1]), ep[k]] = 1
        mass = c @ ind                                   # [t, E] integer
        ep_scores[k] = float(mass.max(axis=1).sum())
        joint[k] = float(mass[np.arange(T), tk[k]].sum())
    tk_scores = None
    if p_ep is not None:
        W = c.astype(np.float64) @ np.asarray(p_ep, dtype=np.float64)
        tk_scores = W[np.arange(T)[None, :], tk].sum(axis=1)
    return ep_scores, tk_scores, joint
