"""Synthetic MoE-layer workloads with controllable expert-affinity skew.

Follows the semantics of the reference's planted-profile generator
(profiles.py:305-376): experts form E = G hidden blocks; a token of planted
cluster c routes to a fixed k-subset of block c with probability 1 - eps and
to k experts of a uniformly chosen other block with probability eps.  Routing
is realised through the gate: hidden states are built so that
top-k(W_g h) is exactly the chosen set, in a fixed order, with a logit margin
far above bf16 rounding, so routing is bit-exact between the GPU and the
fp32 CPU oracle.

Small workloads are generated with numpy (CPU) so the oracle sees the same
bytes; `device=True` builds the big dense tensors on the GPU with torch.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .predictor import DeviceNGramTable, TokenDeviceTable
from .scheduler import LookupBundle

# Public model shapes (external facts, not in the reference): routed experts only.
CONFIGS = {
    "toy": dict(d=256, N=8, k=2, f=512, G=2, vocab=1024),
    "mixtral": dict(d=4096, N=8, k=2, f=14336, G=8, vocab=32000),
    "dsv2_lite": dict(d=2048, N=64, k=6, f=1408, G=8, vocab=102400),
    "qwen2_57b": dict(d=3584, N=64, k=8, f=2560, G=8, vocab=151936),
    # DeepSeek-V2 (the paper's own model): 160 routed experts
    # top-6, hidden 5120, expert ffn 1536 (public config; shared experts are
    # not part of the routed path)
    "deepseek_v2": dict(d=5120, N=160, k=6, f=1536, G=8, vocab=102400),
}


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest bf16 (ties to even), returned as float32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


@dataclass
class Workload:
    cfg: dict
    eps: float
    seed: int
    bundle: LookupBundle
    tokens: np.ndarray                 # int64 [n]
    hist: np.ndarray                   # int64 [n, 2]
    chosen: np.ndarray                 # int64 [n, k] original expert ids, logit order
    gate_w: object                     # [N, d] bf16-valued (np.float32 or torch bf16)
    w1: object                         # [N, f, d]
    w3: object                         # [N, f, d]
    w2: object                         # [N, d, f]
    partials: object                   # [G, n, d]
    expert_labels: np.ndarray = field(default=None)


def make_bundle(G: int, N: int, vocab: int, rng: np.random.Generator, hist_len: int = 2):
    """Lookup tables with the reference's layout (predictor.py:39-82)."""
    npc = N // G
    perm = rng.permutation(N)                       # non-contiguous blocks, as planted
    expert_labels = np.empty(N, dtype=np.int64)
    for c in range(G):
        expert_labels[perm[c * npc:(c + 1) * npc]] = c
    token_labels = rng.integers(0, G, size=vocab).astype(np.int16)
    token_conf = rng.uniform(0.3, 1.0, size=vocab).astype(np.float32)
    rows = G ** hist_len
    counts = np.zeros((rows, G), dtype=np.int64)
    for r in range(rows):
        last = r % G                                 # newest digit
        counts[r, last] = 7
        counts[r] += rng.integers(0, 2, size=G)
    probs = counts / counts.sum(axis=1, keepdims=True)
    tok = TokenDeviceTable(labels=token_labels, confidence=token_conf,
                           provenance=np.zeros(vocab, np.uint8), n_clusters=G)
    ng = DeviceNGramTable(n=hist_len, n_clusters=G, probs=probs, counts=counts)
    return LookupBundle(token_table=tok, ngram_table=ng, expert_labels=expert_labels, layers=1)


def routing_choices(bundle, tokens: np.ndarray, k: int, eps: float, rng) -> np.ndarray:
    """Per occurrence, k distinct original expert ids: the token's preferred
    window inside its planted cluster's block w.p. 1-eps, else a window of
    another block.  When k exceeds the block size (Mixtral EP8: 1 expert per
    cluster) the window continues into the following clusters' blocks."""
    labels = np.asarray(bundle.expert_labels, dtype=np.int64)
    G = int(bundle.token_table.n_clusters)
    blocks = [np.nonzero(labels == c)[0] for c in range(G)]
    cl = np.asarray(bundle.token_table.labels, dtype=np.int64)[tokens]
    n = len(tokens)
    out = np.empty((n, k), dtype=np.int64)
    noisy = rng.random(n) < eps
    other = rng.integers(0, max(G - 1, 1), size=n)
    start = rng.integers(0, 1 << 30, size=n)
    for i in range(n):
        c = int(cl[i])
        if noisy[i] and G > 1:
            c = c + 1 + int(other[i]) % (G - 1)
            s = int(start[i])
        else:
            s = int(tokens[i])                       # fixed preferred window per token
        picked = []
        j = 0
        while len(picked) < k:
            b = blocks[(c + j) % G]
            take = min(k - len(picked), len(b))
            picked.extend(b[(s + np.arange(take)) % len(b)])
            j += 1
        out[i] = picked
    return out


def planted_gate(N: int, d: int, rng) -> np.ndarray:
    """Orthonormal gate rows (bf16-valued float32 [N, d])."""
    q, _ = np.linalg.qr(rng.standard_normal((d, N)))
    return bf16_round(q.T.astype(np.float32))


def planted_partials(gate_w: np.ndarray, chosen: np.ndarray, G: int, rng,
                     alpha: float = 8.0) -> np.ndarray:
    """bf16-valued [G, n, d] attention-TP partials whose reduced rows route,
    through an orthonormal gate, to exactly `chosen` (ordered top-k, original
    expert ids) with logit gaps >= alpha / (2k)."""
    k = chosen.shape[1]
    n, d = chosen.shape[0], gate_w.shape[1]
    coef = (1.0 - 0.5 * np.arange(k) / k).astype(np.float32)
    h = np.float32(alpha) * np.einsum("s,nsd->nd", coef, gate_w[chosen]).astype(np.float32)
    h += 0.05 * rng.standard_normal((n, d)).astype(np.float32)
    z = rng.standard_normal((G, n, d)).astype(np.float32)
    z -= z.mean(0, keepdims=True)
    return bf16_round(h[None] / G + 0.5 * z)


def make_workload(name: str = "toy", n: int = 256, eps: float = 0.1, seed: int = 0,
                  device: bool = False, cfg_override: dict | None = None,
                  hist_consistency: float = 0.9) -> Workload:
    cfg = dict(CONFIGS[name])
    if cfg_override:
        cfg.update(cfg_override)
    G, N, k, d, f, vocab = cfg["G"], cfg["N"], cfg["k"], cfg["d"], cfg["f"], cfg["vocab"]
    if k > N:
        raise ValueError("top_k must not exceed the expert count")
    rng = np.random.default_rng(seed)
    bundle = make_bundle(G, N, vocab, rng)
    tokens = rng.integers(0, vocab, size=n).astype(np.int64)
    cl = np.asarray(bundle.token_table.labels, dtype=np.int64)[tokens]
    hist = rng.integers(0, G, size=(n, 2)).astype(np.int64)
    keep = rng.random(n) < hist_consistency
    hist[keep] = cl[keep, None]
    chosen = routing_choices(bundle, tokens, k, eps, rng)

    # orthonormal gate rows; h = alpha * sum_s c_s w_{chosen_s} + small noise, so
    # logit s of the chosen set is ~alpha*c_s (spacing >= alpha/(2k) = 0.5) and
    # every other logit is ~0: no near-ties anywhere
    q, _ = np.linalg.qr(rng.standard_normal((d, N)))
    wg = bf16_round(q.T.astype(np.float32))
    coef = (1.0 - 0.5 * np.arange(k) / k).astype(np.float32)
    alpha = np.float32(8.0)
    if device:
        import torch
        dev = torch.device("cuda")
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        wg_t = torch.from_numpy(wg).to(dev)
        ch_t = torch.from_numpy(chosen).to(dev)
        h = alpha * (torch.from_numpy(coef).to(dev)[None, :, None] * wg_t[ch_t]).sum(1)
        h += 0.05 * torch.randn((n, d), device=dev, generator=g)
        z = torch.randn((G, n, d), device=dev, generator=g)
        z -= z.mean(0, keepdim=True)
        partials = (h[None] / G + 0.5 * z).to(torch.bfloat16)
        del h, z
        w1 = (torch.randn((N, f, d), device=dev, generator=g) / np.sqrt(d)).to(torch.bfloat16)
        w3 = (torch.randn((N, f, d), device=dev, generator=g) / np.sqrt(d)).to(torch.bfloat16)
        w2 = (torch.randn((N, d, f), device=dev, generator=g) / np.sqrt(f)).to(torch.bfloat16)
        gate_w = wg_t.to(torch.bfloat16)
    else:
        h = alpha * np.einsum("s,nsd->nd", coef, wg[chosen]).astype(np.float32)
        h += 0.05 * rng.standard_normal((n, d)).astype(np.float32)
        z = rng.standard_normal((G, n, d)).astype(np.float32)
        z -= z.mean(0, keepdims=True)
        partials = bf16_round(h[None] / G + 0.5 * z)
        w1 = bf16_round(rng.standard_normal((N, f, d)).astype(np.float32) / np.sqrt(d))
        w3 = bf16_round(rng.standard_normal((N, f, d)).astype(np.float32) / np.sqrt(d))
        w2 = bf16_round(rng.standard_normal((N, d, f)).astype(np.float32) / np.sqrt(f))
        gate_w = wg
    return Workload(cfg=cfg, eps=eps, seed=seed, bundle=bundle, tokens=tokens, hist=hist,
                    chosen=chosen, gate_w=gate_w, w1=w1, w3=w3, w2=w2, partials=partials,
                    expert_labels=np.asarray(bundle.expert_labels, dtype=np.int64))
