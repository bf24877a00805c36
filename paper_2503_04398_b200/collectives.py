"""Standalone shuffled collectives: SRS and SAG (Algorithm 2
lines "RS with shuffle" / "AG with resume").

The reference models these two operators only analytically (comm.py:83-84,
:115); the paper's point is that they replace the attention-TP reduce-scatter
and all-gather of a DS-MoE pipeline at the same cost, with the token
permutation of `rebatch_tokens` / `resume_tokens` riding on the collective.
`SpecMoELayer` runs them fused with the rest of the layer; these entry points
expose them on their own (libsmoe.so `smoe_srs` / `smoe_sag`) for a serving
engine that keeps its own gate and experts:

    tok_s, ix = scheduler.rebatch_tokens(tokens_t, devices_t, G)   # CUDA tensors in
    h = shuffled_reduce_scatter(partials, ix)       # G x [count_g, d]: token group g
    ...                                             # experts on the shuffled groups
    y = shuffled_all_gather(h_out, ix)              # [n, d], original token order

Every partial / block / output is a bf16 CUDA tensor on (or peer-mapped to)
the current device; the sums are fp32 in shard order, rounded once to bf16 —
bit-identical to the layer's SRS.
"""

from __future__ import annotations

import ctypes as C

from . import _dev, _native as N
from .scheduler import SchedulerError, ShuffleIndices


def _plan_tensors(indices: ShuffleIndices):
    t = _dev.torch()
    fwd = indices.forward
    if not (isinstance(fwd, t.Tensor) and fwd.is_cuda):
        fwd = _dev.to_device(fwd, t.int64)
    G, group = int(indices.n_devices), int(indices.group_size)
    fwd = fwd.to(t.int64).contiguous()
    if fwd.numel() < G * group:
        raise SchedulerError("forward index shorter than n_devices * group_size")
    counts = getattr(indices, "_counts_t", None)      # set by rebatch_tokens (device)
    if counts is None or counts.numel() != G:
        counts = (fwd[: G * group].view(G, group) >= 0).sum(1).to(t.int32) if group else \
            t.zeros(G, dtype=t.int32, device=fwd.device)
    group_t = t.full((1,), group, dtype=t.int64, device=fwd.device)
    return fwd, counts, group_t, G, group


def _ptr_array(tensors):
    """Host array of device pointers, passed as one void* (keep it alive)."""
    arr = (C.c_void_p * len(tensors))(*[N.ptr(x) for x in tensors])
    return C.cast(arr, C.c_void_p), arr


def shuffled_reduce_scatter(partials, indices: ShuffleIndices, shards=None):
    """SRS: out_g[j] = bf16( sum_r partials[r][forward[g*group + j]] ), j < count_g.

    partials: G bf16 CUDA tensors [n, d]; indices: the ShuffleIndices of
    `rebatch_tokens`; shards: the token groups to produce (default all, a
    contiguous range).  Returns a list of [count_g, d] tensors."""
    t = _dev.torch()
    fwd, counts, group_t, G, group = _plan_tensors(indices)
    if len(partials) != G:
        raise SchedulerError(f"need {G} partials, got {len(partials)}")
    n, d = int(partials[0].shape[0]), int(partials[0].shape[1])
    for p in partials:
        if p.dtype != t.bfloat16 or not p.is_cuda or tuple(p.shape) != (n, d):
            raise SchedulerError("partials must be bf16 CUDA tensors of one shape [n, d]")
    shards = list(range(G)) if shards is None else list(shards)
    if not shards or shards != list(range(shards[0], shards[0] + len(shards))) \
            or shards[0] < 0 or shards[-1] >= G:
        raise SchedulerError("shards must be a contiguous range of token groups")
    parts = [p.contiguous() for p in partials]
    outs = [t.empty((max(group, 1), d), dtype=t.bfloat16, device=parts[0].device)
            for _ in shards]
    if n:
        (pp, _keep1), (po, _keep2) = _ptr_array(parts), _ptr_array(outs)
        N.check(N.lib().smoe_srs(pp, G, shards[0], len(shards), N.ptr(fwd), N.ptr(counts),
                                 N.ptr(group_t), n, d, po, N.stream_ptr()), "srs")
    c = counts.cpu().tolist()
    return [o[: c[g]] for o, g in zip(outs, shards)]


def shuffled_all_gather(blocks, indices: ShuffleIndices, n_outs: int = 1):
    """SAG: row j of blocks[g] lands at position forward[g*group + j] of the
    [n, d] output (resume_tokens fused with the all-gather).  blocks: G bf16
    CUDA tensors with at least count_g rows.  Returns one [n, d] tensor, or a
    list of n_outs identical copies (one per receiving rank buffer)."""
    t = _dev.torch()
    fwd, counts, group_t, G, group = _plan_tensors(indices)
    if len(blocks) != G:
        raise SchedulerError(f"need {G} blocks, got {len(blocks)}")
    n = int(indices.inverse.shape[0] if hasattr(indices.inverse, "shape")
            else len(indices.inverse))
    d = int(blocks[0].shape[1])
    for b in blocks:
        if b.dtype != t.bfloat16 or not b.is_cuda or int(b.shape[1]) != d:
            raise SchedulerError("blocks must be bf16 CUDA tensors [rows, d]")
    if not 1 <= n_outs <= N.MAX_SHARDS:
        raise SchedulerError("n_outs must be in [1, 16]")
    blks = [b.contiguous() for b in blocks]
    c = counts.cpu().tolist()
    if any(int(b.shape[0]) < c[g] for g, b in enumerate(blks)):
        raise SchedulerError("a block has fewer rows than its token group")
    outs = [t.empty((n, d), dtype=t.bfloat16, device=blks[0].device) for _ in range(n_outs)]
    if n:
        (pb, _keep1), (po, _keep2) = _ptr_array(blks), _ptr_array(outs)
        N.check(N.lib().smoe_sag(pb, G, N.ptr(fwd), N.ptr(counts), N.ptr(group_t), n, d, po,
                                 n_outs, N.stream_ptr()), "sag")
    return outs[0] if n_outs == 1 else outs
