"""DS-MoE pipeline baseline: AR -> A2A -> A2A -> AG (comm.py:99-108).

The comparison point of the north star.  Densely-replicated attention output
is all-reduced on every rank, tokens are sharded by position
(token_dev = i % G, comm.py:202), experts sit in contiguous blocks
(expert_dev = e // (N/G), comm.py:201), and an all-gather restores the batch
on every rank.  Two implementations:

* `DSMoEPipelineLayer` -- the like-for-like baseline.  It runs on the s-MoE
  layer runtime itself (same plan, tcgen05 gate, route, dispatch, grouped
  GEMMs with the combine fused into the down projection, same buffers and
  shard groups), with SMOE_PIPELINE_DSMOE switching the two stages whose
  STRUCTURE differs: a two-shot all-reduce into every process plus each
  rank's slice (instead of the shuffled reduce-scatter), and the combine
  into all-gather blocks plus a resume gather (instead of the fused SAG).
  Position-sharding tables make the plan the DS-MoE one.  s-MoE vs this
  layer therefore differ only in pipeline structure and token placement.
* `DSMoELayer` -- the stock collective pipeline: NCCL all_reduce,
  all_to_all_single with host-synchronised split sizes (x2) and
  all_gather_into_tensor through torch.distributed (one rank per GPU), or,
  with G virtual ranks in one process, the same data movement as device
  copies.  It is the pipeline as DeepSpeed-MoE runs it, kept to exercise
  the NCCL path; it is not the like-for-like comparison.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _native as N
from .layer import SpecMoELayer
from .predictor import DeviceNGramTable, TokenDeviceTable
from .scheduler import LookupBundle


def position_bundle(n_positions: int, n_ranks: int, n_experts: int) -> LookupBundle:
    """Tables under which the s-MoE plan IS the DS-MoE placement: "token"
    (position) i -> rank i % G (comm.py:202) with confidence 1 and no n-gram
    rows, experts in contiguous blocks e // (N/G) (comm.py:201)."""
    G = int(n_ranks)
    if n_experts % G:
        raise ValueError("DS-MoE contiguous placement needs G | N")
    pos = np.arange(int(n_positions))
    tt = TokenDeviceTable(labels=pos % G, confidence=np.ones(len(pos), np.float32),
                          provenance=np.zeros(len(pos), np.uint8), n_clusters=G)
    ng = DeviceNGramTable(n=1, n_clusters=G, probs=np.zeros((G, G)),
                          counts=np.zeros((G, G), np.int64))
    return LookupBundle(token_table=tt, ngram_table=ng,
                        expert_labels=np.arange(n_experts) // (n_experts // G), layers=1)


class DSMoEPipelineLayer(SpecMoELayer):
    """The DS-MoE pipeline on the s-MoE kernels (see the module docstring).

    forward(hidden_partials, n) -> [n, d]: hidden_partials as for
    SpecMoELayer.forward; token ids are the positions 0..n-1."""

    def __init__(self, gate_w, w1, w3, w2, *, n_ranks: int, top_k: int, max_tokens: int,
                 renormalize: bool = True, gate_b=None, group=None, expert_rows=None):
        N_exp = int(np.asarray(gate_w.shape)[0])
        G = int(n_ranks)
        self._ag_rows = G * (-(-int(max_tokens) // G))
        super().__init__(position_bundle(max_tokens, G, N_exp), gate_w, w1, w3, w2,
                         top_k=top_k, max_tokens=max_tokens, renormalize=renormalize,
                         gate_b=gate_b, group=group, expert_rows=expert_rows)
        N.check(self.lib.smoe_layer_set_pipeline(self._h, N.PIPELINE_DSMOE, self._ag_rows),
                "set_pipeline")
        t = _dev.torch()
        self._positions = t.arange(self.max_tokens, dtype=t.int64, device=self.w_gate.device)

    def process_row_buffers(self) -> dict:
        return {"ar": self.max_tokens, "ag": self._ag_rows}

    def stats(self, n: int | None = None) -> dict:
        """As SpecMoELayer.stats, with the DS-MoE collectives' bytes in place
        of the SRS / SAG ones: the two-shot all-reduce moves every token row
        G - 1 times in (reduce-scatter) and G - 1 times out (all-gather), the
        final all-gather G * group rows G - 1 times."""
        st = super().stats(n)
        b = st["bytes"]
        rows = int(sum(st["device_counts"]))
        row = 2 * self.d
        b.pop("srs"), b.pop("sag"), b.pop("srs_padded_model")
        b["all_reduce"] = 2 * (self.G - 1) * rows * row
        b["all_gather"] = (self.G - 1) * self.G * st["group_size"] * row
        return st

    def positions(self, n: int):
        return self._positions[:n]

    def forward(self, hidden_partials, n: int | None = None, out=None):
        hp = hidden_partials
        n = int(hp.shape[-2]) if n is None else int(n)
        return super().forward(hp, self._positions[:n], None, out=out)

    def run_device(self, tokens_t=None, hist_t=None, stream=None, stages=None, hist_depth=None,
                   n: int | None = None):
        if tokens_t is None:
            tokens_t = self._positions[:n]
        return super().run_device(tokens_t, None, stream=stream, stages=stages)


class DSMoELayer:
    def __init__(self, gate_w, w1, w3, w2, *, n_ranks: int, top_k: int, max_tokens: int,
                 renormalize: bool = True, process_group=None, distributed: bool = False):
        t = _dev.torch()
        self.lib = N.lib()
        self.G = int(n_ranks)
        self.k = int(top_k)
        self.max_tokens = int(max_tokens)
        self.renormalize = bool(renormalize)
        self.distributed = distributed
        self.pg = process_group
        gw = _dev.to_device(gate_w, t.bfloat16)
        self.N, self.d = int(gw.shape[0]), int(gw.shape[1])
        self.f = int(w1.shape[1])
        if self.N % self.G:
            raise ValueError("DS-MoE contiguous placement needs G | N")
        self.npc = self.N // self.G
        dev = gw.device
        if distributed:
            import torch.distributed as dist
            self.rank = dist.get_rank(process_group)
            if dist.get_world_size(process_group) != self.G:
                raise ValueError("distributed DS-MoE runs one rank per process")
            self.local_ranks = [self.rank]
        else:
            self.rank = 0
            self.local_ranks = list(range(self.G))
        self.w_gate = gw
        self.owner = t.arange(self.N, device=dev, dtype=t.int32) // self.npc
        self.w13, self.w2 = {}, {}
        for r in self.local_ranks:
            sl = slice(r * self.npc, (r + 1) * self.npc)
            w1r = _dev.to_device(w1[sl] if not isinstance(w1, t.Tensor) else w1[sl], t.bfloat16)
            w3r = _dev.to_device(w3[sl] if not isinstance(w3, t.Tensor) else w3[sl], t.bfloat16)
            packed = t.empty((self.npc, 2 * self.f, self.d), dtype=t.bfloat16, device=dev)
            N.check(self.lib.smoe_pack_w13(N.ptr(w1r.contiguous()), N.ptr(w3r.contiguous()),
                                           self.npc, self.f, self.d, N.ptr(packed),
                                           N.stream_ptr()), "pack_w13")
            self.w13[r] = packed
            self.w2[r] = _dev.to_device(w2[sl] if not isinstance(w2, t.Tensor) else w2[sl],
                                        t.bfloat16).contiguous()
        # the local ranks' experts stacked in rank order: one grouped GEMM covers
        # every resident rank (as SpecMoELayer does for its resident shards)
        self.w13_all = t.cat([self.w13[r] for r in self.local_ranks]).contiguous()
        self.w2_all = t.cat([self.w2[r] for r in self.local_ranks]).contiguous()
        self.w13 = {r: self.w13_all[i * self.npc:(i + 1) * self.npc]
                    for i, r in enumerate(self.local_ranks)}
        self.w2 = {r: self.w2_all[i * self.npc:(i + 1) * self.npc]
                   for i, r in enumerate(self.local_ranks)}
        n, k, d = self.max_tokens, self.k, self.d
        cap = n * k
        self.cap = cap
        L = len(self.local_ranks)
        self.recv_all = t.empty((L, cap, d), dtype=t.bfloat16, device=dev)
        self.hmid_all = t.empty((L, cap, self.f), dtype=t.bfloat16, device=dev)
        self.yrecv_all = t.empty((L, cap, d), dtype=t.bfloat16, device=dev)
        self.buf = {r: {"hs": t.empty((n, d), dtype=t.bfloat16, device=dev),
                        "ids": t.empty((n, k), dtype=t.int32, device=dev),
                        "w": t.empty((n, k), dtype=t.float32, device=dev),
                        "pos": t.empty((n, k), dtype=t.int32, device=dev),
                        "cnt": t.zeros(self.N, dtype=t.int32, device=dev),
                        "send": t.empty((cap, d), dtype=t.bfloat16, device=dev),
                        "recv": self.recv_all[i],
                        "hmid": self.hmid_all[i],
                        "yrecv": self.yrecv_all[i],
                        "yback": t.empty((cap, d), dtype=t.bfloat16, device=dev),
                        "out": t.empty((n, d), dtype=t.bfloat16, device=dev)}
                    for i, r in enumerate(self.local_ranks)}
        self.stats_t = t.zeros(N.STAT_COUNT, dtype=t.int64, device=dev)
        self.problems = t.zeros((512, 4), dtype=t.int64, device=dev)
        self.last = {}

    # ------------------------------------------------------------ collectives
    def _staged(self) -> bool:
        """gloo process groups (tests: several ranks sharing one GPU, where
        NCCL refuses to run) carry the same collectives through host memory;
        NCCL groups run them on the device."""
        import torch.distributed as dist
        return dist.get_backend(self.pg) == "gloo"

    def _all_reduce(self, partials):
        t = _dev.torch()
        if self.distributed:
            import torch.distributed as dist
            if self._staged():
                # fp32 sum in rank order, as the single-process emulation
                h32 = partials[0].float().cpu()
                parts = [t.empty_like(h32) for _ in range(self.G)]
                dist.all_gather(parts, h32, group=self.pg)
                acc = parts[0].clone()
                for p in parts[1:]:
                    acc += p
                return {self.rank: acc.to(t.bfloat16).to(partials[0].device)}
            h = partials[0].clone()
            dist.all_reduce(h, group=self.pg)
            return {self.rank: h}
        import ctypes as C
        n = int(partials[0].shape[0])
        dev = partials[0].device
        h = t.empty_like(partials[0])
        if n:
            # reduce: fp32 sum of the G partials in rank order (the SRS kernel with
            # every token in one group = a plain sum), then the all-gather half:
            # every rank receives the full sum
            fwd = t.arange(n, dtype=t.int64, device=dev)
            counts = t.zeros(self.G, dtype=t.int32, device=dev)
            counts[0] = n
            grp = t.full((1,), n, dtype=t.int64, device=dev)
            parts = [p.contiguous() for p in partials]
            pa = (C.c_void_p * self.G)(*[N.ptr(p) for p in parts])
            po = (C.c_void_p * 1)(N.ptr(h))
            N.check(self.lib.smoe_srs(C.cast(pa, C.c_void_p), self.G, 0, 1, N.ptr(fwd),
                                      N.ptr(counts), N.ptr(grp), n, self.d,
                                      C.cast(po, C.c_void_p), N.stream_ptr()), "all_reduce")
        # every rank holds the sum: co-resident ranks share one copy (as the
        # s-MoE layer's co-resident shards share one SAG output)
        return {r: h for r in self.local_ranks}

    def _gather_counts(self):
        t = _dev.torch()
        if self.distributed:
            import torch.distributed as dist
            if self._staged():
                parts = [t.empty(self.N, dtype=t.int32) for _ in range(self.G)]
                dist.all_gather(parts, self.buf[self.rank]["cnt"].cpu(), group=self.pg)
                return t.stack(parts).numpy().astype(np.int64)
            out = t.empty((self.G, self.N), dtype=t.int32, device=self.w_gate.device)
            dist.all_gather_into_tensor(out, self.buf[self.rank]["cnt"], group=self.pg)
            return out.cpu().numpy().astype(np.int64)
        return t.stack([self.buf[r]["cnt"] for r in range(self.G)]).cpu().numpy().astype(np.int64)

    def _all_to_all(self, name_in, name_out, send_splits, recv_splits):
        """send_splits[r][o] rows go from rank r to rank o; received rows are
        source-major in name_out."""
        t = _dev.torch()
        if self.distributed:
            import torch.distributed as dist
            r = self.rank
            if self._staged():
                # gloo moves no 16-bit types: ship the bf16 rows as bytes
                src = self.buf[r][name_in][: int(sum(send_splits[r]))].view(t.uint8).cpu()
                dst = t.empty((int(sum(recv_splits[r])), 2 * self.d), dtype=t.uint8)
                dist.all_to_all_single(dst, src,
                                       output_split_sizes=[int(x) for x in recv_splits[r]],
                                       input_split_sizes=[int(x) for x in send_splits[r]],
                                       group=self.pg)
                self.buf[r][name_out][: dst.shape[0]].view(t.uint8).copy_(dst)
                return
            dist.all_to_all_single(self.buf[r][name_out][: int(sum(recv_splits[r]))],
                                   self.buf[r][name_in][: int(sum(send_splits[r]))],
                                   output_split_sizes=[int(x) for x in recv_splits[r]],
                                   input_split_sizes=[int(x) for x in send_splits[r]],
                                   group=self.pg)
            return
        soff = {r: np.concatenate([[0], np.cumsum(send_splits[r])]) for r in range(self.G)}
        for o in range(self.G):
            dst = self.buf[o][name_out]
            off = 0
            for r in range(self.G):
                m = int(send_splits[r][o])
                if m:
                    dst[off:off + m].copy_(self.buf[r][name_in][soff[r][o]:soff[r][o] + m])
                off += m

    def _all_gather_out(self, group):
        t = _dev.torch()
        if self.distributed:
            import torch.distributed as dist
            if self._staged():
                mine = self.buf[self.rank]["out"][:group].view(t.uint8).cpu()
                parts = [t.empty_like(mine) for _ in range(self.G)]
                dist.all_gather(parts, mine, group=self.pg)
                return t.cat(parts).to(self.w_gate.device).view(t.bfloat16)
            full = t.empty((self.G * group, self.d), dtype=t.bfloat16, device=self.w_gate.device)
            dist.all_gather_into_tensor(full, self.buf[self.rank]["out"][:group], group=self.pg)
            return full
        return t.cat([self.buf[r]["out"][:group] for r in range(self.G)])

    # ------------------------------------------------------------ forward
    def forward(self, partials, n: int):
        """partials: list (one per local rank) of [n, d] bf16 CUDA tensors.
        Returns the layer output [n, d] in the original token order."""
        t = _dev.torch()
        L, sp = self.lib, N.stream_ptr()
        G, k, d, npc = self.G, self.k, self.d, self.npc
        dev = self.w_gate.device
        # 1. all-reduce of the attention-TP partials
        H = self._all_reduce(partials)
        # 2. position sharding plan (comm.py:202: token i -> rank i % G)
        devices = t.arange(n, device=dev, dtype=t.int64) % G
        fwd = t.empty(G * max(n, 1), dtype=t.int64, device=dev)
        inv = t.empty(n, dtype=t.int64, device=dev)
        counts = t.empty(G, dtype=t.int32, device=dev)
        group_t = t.empty(1, dtype=t.int64, device=dev)
        ws_b = int(L.smoe_plan_workspace_bytes(n, G))
        ws = t.empty(ws_b, dtype=t.uint8, device=dev)
        N.check(L.smoe_rebatch_plan(N.ptr(devices), n, G, N.ptr(fwd), N.ptr(inv), N.ptr(counts),
                                    N.ptr(group_t), 0, N.ptr(ws), ws_b, sp), "plan")
        cnt_h = [(n - r + G - 1) // G for r in range(G)]            # i % G sharding
        group = max(cnt_h) if n else 0
        self.stats_t.zero_()
        for r in self.local_ranks:
            b = self.buf[r]
            rows = cnt_h[r]
            idx = fwd[r * group: r * group + rows]
            # 3. my token rows
            N.check(L.smoe_gather_rows(N.ptr(H[r]), n, 2, d, N.ptr(idx), rows, 0, 0, N.ptr(b["hs"]),
                                       0, sp), "gather")
            # 4. gate + 5. expert-major send positions + 6. pack
            N.check(L.smoe_gate_topk(N.ptr(b["hs"]), rows, d, N.ptr(self.w_gate), 0, self.N, k,
                                     int(self.renormalize), N.ptr(self.owner), r, N.ptr(b["ids"]),
                                     N.ptr(b["w"]), N.ptr(self.stats_t), sp), "gate")
            N.check(L.smoe_pair_offsets(N.ptr(b["ids"]), rows, k, self.N, N.ptr(b["pos"]),
                                        N.ptr(b["cnt"]), sp), "pair_offsets")
            N.check(L.smoe_pack_rows(N.ptr(b["hs"]), rows, k, d, N.ptr(b["pos"]), N.ptr(b["send"]),
                                     sp), "pack")
        # 7. counts exchange (host sync: all2allv needs split sizes)
        C = self._gather_counts()                                # [G src, N]
        send = {r: [int(C[r, o * npc:(o + 1) * npc].sum()) for o in range(G)] for r in range(G)}
        recv = {o: [send[r][o] for r in range(G)] for o in range(G)}
        # 8. dispatch all-to-all
        self._all_to_all("send", "recv", send, recv)
        # 9. experts: ONE grouped GEMM over every local rank, problems =
        #    (local rank o, source rank r, expert of o) in o's source-major rows
        probs = []
        for i, o in enumerate(self.local_ranks):
            off = 0
            for r in range(G):
                for e in range(o * npc, (o + 1) * npc):
                    m = int(C[r, e])
                    probs.append([i * self.cap + off, m, i * npc + (e - o * npc),
                                  i * self.cap + off])
                    off += m
        if len(probs) > self.problems.shape[0]:
            raise ValueError("too many (rank, source, expert) problems for one launch")
        if probs:
            self.problems[: len(probs)].copy_(t.as_tensor(probs, dtype=t.int64))
            La = len(self.local_ranks)
            N.check(L.smoe_grouped_gemm(N.ptr(self.recv_all), La * self.cap, d,
                                        N.ptr(self.w13_all), La * npc * 2 * self.f, 2 * self.f,
                                        N.ptr(self.problems), len(probs), 1,
                                        N.ptr(self.hmid_all), La * self.cap, self.f, sp), "gemm_up")
            N.check(L.smoe_grouped_gemm(N.ptr(self.hmid_all), La * self.cap, self.f,
                                        N.ptr(self.w2_all), La * npc * d, d, N.ptr(self.problems),
                                        len(probs), 0, N.ptr(self.yrecv_all), La * self.cap, d,
                                        sp), "gemm_down")
        # 10. combine all-to-all (reverse splits)
        self._all_to_all("yrecv", "yback", recv, send)
        # 11. weighted combine of the k expert outputs
        for r in self.local_ranks:
            b = self.buf[r]
            N.check(L.smoe_combine_rows(N.ptr(b["yback"]), N.ptr(b["pos"]), N.ptr(b["w"]),
                                        cnt_h[r], k, d, N.ptr(b["out"]), sp), "combine")
        # 12. all-gather and restore the original order
        full = self._all_gather_out(group)
        out = t.empty((n, d), dtype=t.bfloat16, device=dev)
        N.check(L.smoe_gather_rows(N.ptr(full), full.shape[0], 2, d, N.ptr(inv), n, 0, 0,
                                   N.ptr(out), 0, sp), "resume")
        self.last = {"counts": C, "group": group, "send_splits": send}
        return out

    def stats(self) -> dict:
        s = self.stats_t.cpu().numpy()
        loc, rem = int(s[0]), int(s[1])
        row = 2 * self.d
        return {"local_tokens": loc, "remote_tokens": rem,
                "measured_alpha": loc / max(loc + rem, 1),
                "bytes": {"all_reduce": None, "a2a_dispatch": rem * row, "a2a_combine": rem * row}}
