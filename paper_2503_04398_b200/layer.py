"""The speculative-token-shuffling MoE layer (Algorithm 2).

`SpecMoELayer(bundle, gate_w, w1, w3, w2, ...)` takes the offline solver's
E/T/S tables (a `LookupBundle`, scheduler.py:24-38) and the expert weights in
the ORIGINAL expert order, applies the s-EG placement (gate_permutation,
scheduler.py:200-210) once at construction, and runs the forward:

    plan (lookup + stable partition) -> SRS -> gate/top-k -> route ->
    A2A dispatch (local pairs stay local) -> SwiGLU grouped GEMM (tcgen05) ->
    down GEMM whose epilogue writes the A2A combine -> weighted combine + SAG

G shards ("virtual ranks", G = the bundle's cluster count) are resident in
this process; with a `ShardGroup` (dist.py) they are spread over processes /
GPUs and the peer buffers are CUDA-IPC mappings.  Every stage is one or two
kernels of libsmoe.so; there is no CPU fallback.

Data layout in HBM (per shard g unless noted; n = max_tokens, k = top_k):
    partial[g]  bf16 [n, d]        attention-TP partial sum (input)
    hs[g]       bf16 [n, d]        SRS output, rows of group g in slot order
    topk ids/w  i32/f32 [n, k]     s-EG expert slot and combine weight
    xin[g]      bf16 [R, d]        expert-major input rows (R = expert_rows)
    hmid        bf16 [L*R, f]      SwiGLU activations (L resident shards)
    ypair[g]    bf16 [n*k, d]      expert output per (token, k-slot)
    out[g]      bf16 [n, d]        layer output in original token order
"""

from __future__ import annotations

import numpy as np

from . import _dev, _native
from .scheduler import LookupBundle, SchedulerError, device_tables, gate_permutation

N = _native


class SpecMoELayer:
    def __init__(self, bundle, gate_w, w1, w3, w2, *, top_k: int, max_tokens: int,
                 gate_b=None, renormalize: bool = True, expert_rows: int | None = None,
                 group=None, shared_from: "SpecMoELayer | None" = None):
        """shared_from: another layer whose s-EG-ordered weights this one
        reuses (no copy, no repacking) -- micro-batches of one layer."""
        t = _dev.torch()
        self.lib = N.lib()
        self.bundle = bundle
        self.G = int(bundle.token_table.n_clusters)
        if self.G > N.MAX_SHARDS:
            raise SchedulerError(f"{self.G} shards exceed the supported {N.MAX_SHARDS}")
        gate_w = _dev.to_device(gate_w, t.bfloat16)
        self.N, self.d = int(gate_w.shape[0]), int(gate_w.shape[1])
        self.f = int((shared_from.f if shared_from is not None else w1.shape[1]))
        self.k = int(top_k)
        self.max_tokens = int(max_tokens)
        self.expert_rows = int(expert_rows or self.max_tokens * self.k)
        self.renormalize = bool(renormalize)
        labels = np.asarray(bundle.expert_labels, dtype=np.int64)
        if len(labels) != self.N:
            raise SchedulerError("expert labels do not match the gate width")
        self.group = group
        world = group.world_size if group else 1
        rank = group.rank if group else 0
        if self.G % world:
            raise SchedulerError("shards must divide evenly over processes")
        spp = self.G // world
        self.shard_begin, self.shard_count = rank * spp, spp
        self.world, self.rank = world, rank

        if shared_from is not None:
            src = shared_from
            for a in ("perm", "slot_owner", "slot_first", "local_slots", "w_gate", "b_gate",
                      "w13", "w2", "w_tiled"):
                setattr(self, a, getattr(src, a))
        else:
            self._place_weights(labels, gate_w, gate_b, w1, w3, w2)
        self.tables = device_tables(bundle)
        self._alloc_buffers()
        self._create_handle()

    def _place_weights(self, labels, gate_w, gate_b, w1, w3, w2):
        """s-EG placement (scheduler.py:200-224), computed on the GPU, and the
        resident experts' weights in slot order."""
        t = _dev.torch()
        self.perm = gate_permutation(labels, self.G)
        n2o = np.asarray(self.perm.new_to_old)
        self.slot_owner = labels[n2o].astype(np.int32)          # cluster of each slot
        first = np.searchsorted(self.slot_owner, np.arange(self.G + 1), side="left")
        self.slot_first = first.astype(np.int64)
        e0 = int(first[self.shard_begin])
        e1 = int(first[self.shard_begin + self.shard_count])
        self.local_slots = e1 - e0
        if self.local_slots > 256:
            raise SchedulerError("more than 256 resident experts per process")
        n2o_t = t.as_tensor(n2o, device=gate_w.device)
        self.w_gate = gate_w.index_select(0, n2o_t).contiguous()
        self.b_gate = None
        if gate_b is not None:
            self.b_gate = _dev.to_device(gate_b, t.float32).index_select(0, n2o_t).contiguous()
        local_ids = n2o_t[e0:e1]
        w1l = _dev.to_device(w1, t.bfloat16).index_select(0, local_ids).contiguous()
        w3l = _dev.to_device(w3, t.bfloat16).index_select(0, local_ids).contiguous()
        self.w2 = _dev.to_device(w2, t.bfloat16).index_select(0, local_ids).contiguous()
        self.w13 = t.empty((max(self.local_slots, 1), 2 * self.f, self.d), dtype=t.bfloat16,
                           device=gate_w.device)
        if self.local_slots:
            N.check(self.lib.smoe_pack_w13(N.ptr(w1l), N.ptr(w3l), self.local_slots, self.f,
                                           self.d, N.ptr(self.w13), N.stream_ptr()), "pack_w13")
        del w1l, w3l
        # box-tiled copies: every 256 x 64 weight box the GEMMs load is one
        # contiguous 32 KiB run (SMOE_UNTILED_WEIGHTS=1 keeps row-major, A/B only)
        import os
        self.w_tiled = bool(self.local_slots) and os.environ.get("SMOE_UNTILED_WEIGHTS") != "1"
        if self.w_tiled:
            for name, rows, cols in (("w13", self.local_slots * 2 * self.f, self.d),
                                     ("w2", self.local_slots * self.d, self.f)):
                src = getattr(self, name)
                dst = t.empty_like(src)
                N.check(self.lib.smoe_tile_weights(N.ptr(src), rows, cols, N.ptr(dst),
                                                   N.stream_ptr()), "tile_weights")
                setattr(self, name, dst)
                del src

    # ------------------------------------------------------------ buffers
    def process_row_buffers(self) -> dict:
        """Extra per-process [rows, d] bf16 peer buffers {name: rows} bound to
        the C slots of `_EXTRA_SLOTS` (none for the speculative pipeline)."""
        return {}

    _EXTRA_SLOTS = {"ar": N.BUF_AR, "ag": N.BUF_AG}

    def _alloc_buffers(self):
        t = _dev.torch()
        dev = self.w_gate.device
        G, L, n, d, k, f, R = (self.G, self.shard_count, self.max_tokens, self.d, self.k,
                               self.f, self.expert_rows)
        bf = t.bfloat16
        if self.group is None:
            self.partial = t.zeros((G, n, d), dtype=bf, device=dev)
            self.xin = t.empty((G, R, d), dtype=bf, device=dev)
            self.xmeta = t.empty((G, R), dtype=t.int64, device=dev)
            self.ypair = t.empty((G, n * k, d), dtype=bf, device=dev)
            self.out_buf = t.empty((n, d), dtype=bf, device=dev)
            self.counts_mat = t.zeros((G, self.N), dtype=t.int32, device=dev)
            self.hist_next = t.zeros((n, max(self.tables.ngram_n, 1)), dtype=t.int64, device=dev)
            peer = {"partial": [self.partial[g] for g in range(G)],
                    "xin": [self.xin[g] for g in range(G)],
                    "xmeta": [self.xmeta[g] for g in range(G)],
                    "ypair": [self.ypair[g] for g in range(G)],
                    "out": [self.out_buf] * G,         # one copy per process (SAG)
                    "counts": [self.counts_mat] * G,
                    "hist": [self.hist_next] * G,
                    "signal": [None] * G}
            for name, rows in self.process_row_buffers().items():
                buf = t.empty((rows, d), dtype=bf, device=dev)
                peer[name] = [buf] * G
                peer[name + "_local"] = buf
        else:
            peer = self.group.alloc_layer_buffers(self, dev)
            self.partial = peer["partial_local"]
            self.out_buf = peer["out_local"]
            self.counts_mat = peer["counts_local"]
            self.hist_next = peer["hist_local"]
        self._peer = peer
        for name in self.process_row_buffers():
            setattr(self, name + "_local", peer[name + "_local"])
        # every resident shard's output is the process's single output buffer
        # (indexable per shard for the reference-style per-rank view)
        self.out = self.out_buf.unsqueeze(0).expand(G if self.group is None else L, n, d)
        self.hs = t.empty((L, n, d), dtype=bf, device=dev)
        self.topk_ids = t.empty((L, n, k), dtype=t.int32, device=dev)
        self.topk_w = t.empty((L, n, k), dtype=t.float32, device=dev)
        self.pair_rank = t.empty((L, n, k), dtype=t.int32, device=dev)
        self.hmid = t.empty((L * R, f), dtype=bf, device=dev)
        # Rows of a 128-row GEMM tile past an expert's routed rows are whatever
        # the expert-input / hidden buffers hold, and the MMA rate depends on
        # operand values: at decode sizes the DSV2-Lite up GEMM takes 163 us
        # over zeros (a fresh allocation) or large values, 122 us over small
        # noise (profiles/r1_gemm_l2/decode_padding_fill_scan.csv).  Start
        # them as small noise; those rows are never stored, so no result
        # depends on it.
        gen = t.Generator(device=dev).manual_seed(0)
        (self.xin if self.group is None else peer["xin_local"]).normal_(0.0, 0.01, generator=gen)
        self.hmid.normal_(0.0, 0.01, generator=gen)
        self.forward_buf = t.empty(G * n, dtype=t.int64, device=dev)
        self.inverse = t.empty(n, dtype=t.int64, device=dev)
        self.dev = t.empty(n, dtype=t.int64, device=dev)
        self.plan_counts = t.zeros(G, dtype=t.int32, device=dev)
        self.group_t = t.zeros(1, dtype=t.int64, device=dev)
        self.stats_t = t.zeros(N.STAT_COUNT, dtype=t.int64, device=dev)
        self.err = t.zeros(1, dtype=t.int32, device=dev)
        self.problems = t.zeros((256, 4), dtype=t.int64, device=dev)
        self.epoch = t.zeros(1, dtype=t.int32, device=dev)

    def _create_handle(self):
        cfg = N.LayerConfig(n_shards=self.G, shard_begin=self.shard_begin,
                            shard_count=self.shard_count, n_experts=self.N, top_k=self.k,
                            hidden=self.d, ffn=self.f, renormalize=int(self.renormalize),
                            max_tokens=self.max_tokens, expert_rows=self.expert_rows,
                            world_size=self.world, world_rank=self.rank)
        import ctypes as C
        self._cfg = cfg
        ws_bytes = int(self.lib.smoe_layer_workspace_bytes(C.byref(cfg)))
        t = _dev.torch()
        self.workspace = t.empty(max(ws_bytes, 256), dtype=t.uint8, device=self.w_gate.device)
        h = C.c_void_p()
        N.check(self.lib.smoe_layer_create(C.byref(cfg), C.byref(h)), "layer_create")
        self._h = h
        bind = lambda slot, i, x: N.check(  # noqa: E731
            self.lib.smoe_layer_bind(h, slot, i, 0 if x is None else N.ptr(x) if
                                     hasattr(x, "data_ptr") else int(x)), "layer_bind")
        p = self._peer
        for g in range(self.G):
            bind(N.BUF_PARTIAL, g, p["partial"][g])
            bind(N.BUF_XIN, g, p["xin"][g])
            bind(N.BUF_XMETA, g, p["xmeta"][g])
            if "xfan" in p:                     # processes > 1: deduplicated dispatch
                bind(N.BUF_XFAN, g, p["xfan"][g])
            bind(N.BUF_YPAIR, g, p["ypair"][g])
            bind(N.BUF_OUT, g, p["out"][g])
            bind(N.BUF_COUNTS, g, p["counts"][g])
            bind(N.BUF_HIST_OUT, g, p["hist"][g])
            if p["signal"][g] is not None:
                bind(N.BUF_SIGNAL, g, p["signal"][g])
            for name in self.process_row_buffers():
                bind(self._EXTRA_SLOTS[name], g, p[name][g])
        for i in range(self.shard_count):
            bind(N.BUF_HS, i, self.hs[i])
            bind(N.BUF_TOPK_IDS, i, self.topk_ids[i])
            bind(N.BUF_TOPK_W, i, self.topk_w[i])
            bind(N.BUF_PAIR_RANK, i, self.pair_rank[i])
        for slot, x in ((N.BUF_HMID, self.hmid), (N.BUF_FORWARD, self.forward_buf),
                        (N.BUF_INVERSE, self.inverse), (N.BUF_DEV, self.dev),
                        (N.BUF_PLAN_COUNTS, self.plan_counts), (N.BUF_GROUP, self.group_t),
                        (N.BUF_STATS, self.stats_t), (N.BUF_ERR, self.err),
                        (N.BUF_WORKSPACE, self.workspace), (N.BUF_PROBLEMS, self.problems),
                        (N.BUF_EPOCH, self.epoch)):
            bind(slot, 0, x)
        tb = self.tables
        owner = (C.c_int32 * self.N)(*[int(x) for x in self.slot_owner])
        N.check(self.lib.smoe_layer_set_tables(
            h, N.ptr(tb.t_labels), N.ptr(tb.t_conf), tb.vocab, N.ptr(tb.a_best), N.ptr(tb.a_conf),
            tb.a_rows, tb.ngram_n, owner), "layer_set_tables")
        set_w = (self.lib.smoe_layer_set_weights_tiled if self.w_tiled
                 else self.lib.smoe_layer_set_weights)
        N.check(set_w(h, N.ptr(self.w_gate), N.ptr(self.b_gate), N.ptr(self.w13), N.ptr(self.w2)),
                "layer_set_weights")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self.lib.smoe_layer_destroy(h)
            except Exception:
                pass

    # ------------------------------------------------------------ forward
    def partial_views(self, n: int):
        """[L, n, d] views of the resident shards' partial-input buffers
        currently bound to the layer (write the attention-TP partials here to
        avoid a copy)."""
        return getattr(self, "_bound_partial", self.partial)[:, :n]

    def _bind_partial(self, P, peer_ptrs=None):
        """Bind the partial-input buffers: P is this process's [L, n, d] view;
        peer_ptrs the G per-shard addresses (every process's copy of the same
        slot) when shards span processes."""
        if getattr(self, "_bound_partial", self.partial) is P:
            return
        for g in range(self.G):
            ptr = N.ptr(P[g]) if peer_ptrs is None else int(peer_ptrs[g])
            N.check(self.lib.smoe_layer_bind(self._h, N.BUF_PARTIAL, g, ptr), "bind")
        self._bound_partial = P

    @property
    def history_width(self) -> int:
        """Digits of the n-gram window (the bundle's n, predictor.py:57-82)."""
        return int(self.tables.ngram_n)

    def _device_inputs(self, tokens_t, hist_t, hist_depth, max_tokens=None):
        """Validated, contiguous int64 device views of the token ids and the
        history window, and the window's valid depth.  The kernels index the
        window as [n, history_width] with a fixed stride, so any other shape
        is rejected (IndexError, as numpy raises for rows outside the n-gram
        table) instead of being misread."""
        t = _dev.torch()
        dev = self.w_gate.device
        tok = tokens_t.reshape(-1).to(device=dev, dtype=t.int64).contiguous()
        n = int(tok.shape[0])
        cap = self.max_tokens if max_tokens is None else int(max_tokens)
        if n > cap:
            raise SchedulerError(f"{n} tokens exceed max_tokens={cap}")
        if hist_t is None:
            return tok, None, 0
        h = self.history_width
        if hist_t.dim() != 2 or tuple(hist_t.shape) != (n, h):
            raise IndexError(f"histories must be [{n}, {h}] (tokens x n-gram depth), "
                             f"got {tuple(hist_t.shape)}")
        depth = h if hist_depth is None else int(hist_depth)
        if not 0 <= depth <= h:
            raise ValueError(f"history_depth must be in [0, {h}]")
        hist = hist_t.to(device=dev, dtype=t.int64).contiguous()
        return tok, hist, depth

    def run_device(self, tokens_t, hist_t=None, stream=None, stages=None, hist_depth=None):
        """Run the layer on device-resident inputs already in the partial
        buffers; no host synchronisation (graph-capturable).

        hist_t: [n, history_width] window of the previous layers' top-1
        clusters or None (first layer); hist_depth: how many of its newest
        digits are valid (default: all).  The n-gram lookup is used only for
        a full window, as the reference passes histories=None for the first
        n layers (scheduler.py:84-89)."""
        tok, hist, depth = self._device_inputs(tokens_t, hist_t, hist_depth)
        n = int(tok.shape[0])
        self._inputs = (tok, hist)                 # alive until the kernels ran
        sp = N.stream_ptr(stream)
        hp = N.ptr(hist)
        w = self.history_width
        if stages is None:
            N.check(self.lib.smoe_layer_forward_hist(self._h, N.ptr(tok), hp, w, depth, n, sp),
                    "layer_forward")
        else:
            for s in stages:
                N.check(self.lib.smoe_layer_stage_hist(self._h, s, N.ptr(tok), hp, w, depth,
                                                       n, sp),
                        f"layer stage {N.STAGE_NAMES[s]}")
        if stages is None or N.STAGE_COMBINE_SAG in stages:
            self._hist_depth_out = min(depth + 1, w)
        return self.out_view(n)

    def tune_gemm_order(self, tokens_t, hist_t=None, candidates=((1, 0), (2, -2)),
                        rounds: int = 4, reps: int = 2) -> dict:
        """Pick the up GEMM's schedule -- (cta_group, tile order) -- for this
        batch on this GPU by interleaved timing (ABBA rounds) of whole
        forwards, set it process-wide (SMOE_OPT_GEMM_CTA_GROUP_UP /
        SMOE_OPT_GEMM_GROUP_M_UP) and return the timings.  Every schedule
        gives bit-identical outputs; which one is faster depends on the GPU
        (under the power cap the SM pair's fewer shared-memory bytes per flop
        trade against its L2 misses, profiles/r2/gemm_cg_up/).  Decode-sized
        batches always run one SM per tile: nothing to tune there."""
        t = _dev.torch()
        lib = self.lib
        n = int(t.as_tensor(tokens_t).reshape(-1).shape[0])
        pair_min = lib.smoe_get_option(N.OPT_GEMM_PAIR_MIN_ROWS)
        cur = (lib.smoe_get_option(N.OPT_GEMM_CTA_GROUP_UP),
               lib.smoe_get_option(N.OPT_GEMM_GROUP_M_UP))
        if n * self.k <= pair_min * self.N:
            return {"choice": list(cur), "tuned": False}

        def use(c):
            N.check(lib.smoe_set_option(N.OPT_GEMM_CTA_GROUP_UP, int(c[0])), "opt")
            N.check(lib.smoe_set_option(N.OPT_GEMM_GROUP_M_UP, int(c[1])), "opt")

        ms = {c: [] for c in candidates}
        for c in candidates:                      # warm each schedule (maps, caches)
            use(c)
            self.run_device(tokens_t, hist_t)
        t.cuda.synchronize()
        for r in range(rounds):
            order = list(candidates) if r % 2 == 0 else list(reversed(candidates))
            for c in order:
                use(c)
                self.run_device(tokens_t, hist_t)
                e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    self.run_device(tokens_t, hist_t)
                e1.record()
                t.cuda.synchronize()
                ms[c].append(e0.elapsed_time(e1) / reps)
        med = {c: sorted(v)[len(v) // 2] for c, v in ms.items()}
        best = min(candidates, key=lambda c: med[c])
        use(best)
        self.check_errors()
        return {"choice": list(best), "tuned": True,
                "median_ms": {f"cg{c[0]}_gm{c[1]}": round(v, 4) for c, v in med.items()}}

    def capture(self, tokens_t, hist_t=None, hist_depth=None):
        """Record one forward over these device tensors as a CUDA graph.

        Replaying the returned `torch.cuda.CUDAGraph` re-runs the whole layer
        (every stage, one graph launch) on whatever the bound partial buffers,
        `tokens_t` and `hist_t` hold at replay time; the token count is fixed
        at capture.  For small (decode-sized) batches, where the ten kernel
        launches of `run_device` cost as much as the work.  With a ShardGroup
        every process captures and replays in lockstep: the signal-pad barriers
        count epochs in device memory, so replays stay ordered across processes."""
        t = _dev.torch()
        # the graph reads these exact buffers at replay: they must already be
        # contiguous int64 device tensors (no hidden copy inside the capture)
        for x in (tokens_t, hist_t):
            if x is not None and not (x.is_cuda and x.dtype == t.int64 and x.is_contiguous()):
                raise ValueError("capture() needs contiguous int64 CUDA token ids / histories")
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(s):                  # warm-up off the capture (lazy attributes)
            self.run_device(tokens_t, hist_t, stream=s, hist_depth=hist_depth)
        t.cuda.current_stream().wait_stream(s)
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g):
            self.run_device(tokens_t, hist_t, hist_depth=hist_depth)
        return g

    def out_view(self, n: int, shard: int | None = None):
        g = self.shard_begin if shard is None else shard
        if self.group is None:
            return self.out[g, :n]
        return self.out[g - self.shard_begin, :n]

    def next_history(self, n: int):
        """[n, h] device view of the n-gram window for the NEXT MoE layer,
        written by the last forward: the input window shifted by one layer
        plus the cluster of each token's top-1 expert (predictor.py:165-166),
        or None while fewer than h layers of routing have been observed --
        the reference's contract is histories=None for the first n layers
        (scheduler.py:84-89).  `history_window` returns the partial window."""
        win, depth = self.history_window(n)
        return win if depth >= self.history_width and depth > 0 else None

    def history_window(self, n: int):
        """(window [n, h] device view, valid depth): the next layer's n-gram
        window and how many of its newest digits are real top-1 clusters.
        Chain layers with `forward(..., histories=win, history_depth=depth)`;
        the lookup switches to the n-gram table once depth == h."""
        return self.hist_next[:n], int(getattr(self, "_hist_depth_out", 0))

    def forward(self, hidden_partials, token_ids, histories=None, out=None,
                history_depth=None):
        """Full layer from user tensors (host or device).

        hidden_partials: [L, n, d] (one partial per resident shard) or [n, d]
        when there is a single shard; token_ids int [n]; histories int [n, h]
        (h = the bundle's n-gram depth) or None; history_depth: valid newest
        digits of `histories` (default h, see `history_window`).
        Returns the layer output [n, d] (bf16) in the original token order:
        a device view for CUDA inputs, else a host tensor (`out` if given —
        pass pinned host tensors for asynchronous copies).
        """
        t = _dev.torch()
        host = not (isinstance(hidden_partials, t.Tensor) and hidden_partials.is_cuda)

        def dev_i64(x):
            if isinstance(x, t.Tensor):
                return x.to(device=self.w_gate.device, dtype=t.int64,
                            non_blocking=True).contiguous()
            return _dev.to_device(np.ascontiguousarray(x), t.int64)

        tok = dev_i64(token_ids).reshape(-1)
        n = int(tok.numel())
        if n > self.max_tokens:
            raise SchedulerError(f"{n} tokens exceed max_tokens={self.max_tokens}")
        hist = None if histories is None else dev_i64(histories)
        self._device_inputs(tok, hist, history_depth)      # validate before any copy
        hp = hidden_partials if isinstance(hidden_partials, t.Tensor) else t.as_tensor(
            np.asarray(hidden_partials))
        if hp.dim() == 2:
            hp = hp.unsqueeze(0)
        if hp.shape[0] != self.shard_count or hp.shape[1] != n or hp.shape[2] != self.d:
            raise SchedulerError(f"partials must be [{self.shard_count}, {n}, {self.d}]")
        dst = self.partial_views(n)
        if hp.dtype == t.bfloat16:
            dst.copy_(hp, non_blocking=True)
        else:
            dst.copy_(hp.to(device=dst.device, non_blocking=True).to(t.bfloat16))
        res = self.run_device(tok, hist, hist_depth=history_depth)
        if not host:
            self.check_errors()
            return res
        if out is None:
            out = t.empty((n, self.d), dtype=t.bfloat16)
        out.copy_(res, non_blocking=out.is_pinned())
        self.check_errors()                 # stream sync: `out` is complete after this
        return out

    # ------------------------------------------------------------ pipelined serving
    def forward_async(self, hidden_partials, token_ids, histories=None, out=None,
                      history_depth=None):
        """Pipelined `forward` for a stream of batches from HOST memory.

        Returns a handle whose `.result()` yields the host output.  Inputs
        should be pinned CPU tensors (their H2D copy runs on a copy stream);
        `out` a pinned [n, d] bf16 tensor.  Partials are double-buffered:
        the H2D of batch i+1 overlaps the layer of batch i (the buffer is
        released as soon as batch i's SRS has read it), and the D2H of batch
        i overlaps the first stages of batch i+1.  With shards spread over
        processes (a ShardGroup) both partial slots are peer-visible and every
        process must issue the same sequence of batches.  Data-dependent
        errors of a batch surface in its own `.result()`, which waits for
        that batch's D2H only (never drains the compute stream, so the H2D
        of the next batch is already queued behind the running one).
        """
        t = _dev.torch()
        n = int(token_ids.shape[0])
        if n > self.max_tokens:
            raise SchedulerError(f"{n} tokens exceed max_tokens={self.max_tokens}")
        hp = hidden_partials if hidden_partials.dim() == 3 else hidden_partials.unsqueeze(0)
        if tuple(hp.shape) != (self.shard_count, n, self.d) or hp.dtype != t.bfloat16:
            raise SchedulerError(f"partials must be bf16 [{self.shard_count}, {n}, {self.d}]")
        if histories is not None and tuple(histories.shape) != (n, self.history_width):
            raise IndexError(f"histories must be [{n}, {self.history_width}]")
        if token_ids.dim() != 1:
            raise SchedulerError("token_ids must be 1-D")
        # every input is validated before the pipeline state moves: a rejected
        # batch must not flip the slot parity (peers in a ShardGroup follow
        # the same batch sequence and barrier epochs)
        st = self._pipeline()
        i = st["count"]
        st["count"] += 1
        slot = i % 2
        P, tok, hist = st["P"][slot], st["tok"][slot], st["hist"][slot]
        # ---- H2D on the copy stream, once the slot's previous batch has passed its SRS
        with t.cuda.stream(st["h2d"]):
            st["h2d"].wait_event(st["free_p"][slot])     # batch i-2 finished its SRS
            P[:, :n].copy_(hp, non_blocking=True)
            st["h2d"].wait_event(st["free_ids"][slot])   # batch i-2 finished the layer
            tok[:n].copy_(token_ids, non_blocking=True)
            if histories is not None:
                hist[:n].copy_(histories, non_blocking=True)
            st["in"][slot].record(st["h2d"])
        # ---- the layer on the compute stream
        cs = st["compute"]
        self._bind_partial(P, st["peer_P"][slot])
        with t.cuda.stream(cs):
            cs.wait_event(st["in"][slot])
            hp_t = hist[:n] if histories is not None else None
            if self.group is None:
                self.run_device(tok[:n], hp_t, stream=cs, hist_depth=history_depth,
                                stages=[N.STAGE_PLAN, N.STAGE_SRS])
                st["free_p"][slot].record(cs)
                self.run_device(tok[:n], hp_t, stream=cs, hist_depth=history_depth,
                                stages=range(N.STAGE_GATE, N.STAGE_COMBINE_SAG))
                cs.wait_event(st["d2h_done"])      # previous output fully read out
                self.run_device(tok[:n], hp_t, stream=cs, hist_depth=history_depth,
                                stages=[N.STAGE_COMBINE_SAG])
            else:
                # peers read this process's partial slot in their SRS and write
                # its output buffer in their SAG: the slot is free once every
                # process passed this batch's ROUTE barrier, and the previous
                # D2H must end before the barrier that closes EXPERT_DOWN
                self.run_device(tok[:n], hp_t, stream=cs, hist_depth=history_depth,
                                stages=range(N.STAGE_PLAN, N.STAGE_DISPATCH))
                st["free_p"][slot].record(cs)
                self.run_device(tok[:n], hp_t, stream=cs, hist_depth=history_depth,
                                stages=[N.STAGE_DISPATCH, N.STAGE_EXPERT_UP])
                cs.wait_event(st["d2h_done"])
                self.run_device(tok[:n], hp_t, stream=cs, hist_depth=history_depth,
                                stages=[N.STAGE_EXPERT_DOWN, N.STAGE_COMBINE_SAG])
            # this batch's error flag, read out before the next batch's plan
            # resets it (stream order); the host reads it in .result()
            err = t.empty(1, dtype=t.int32, pin_memory=True)
            err.copy_(self.err, non_blocking=True)
            st["free_ids"][slot].record(cs)
            st["done"].record(cs)
        # ---- D2H on its own stream
        if out is None:
            out = t.empty((n, self.d), dtype=t.bfloat16, pin_memory=True)
        ev = t.cuda.Event()
        with t.cuda.stream(st["d2h"]):
            st["d2h"].wait_event(st["done"])
            out.copy_(self.out_view(n), non_blocking=True)
            st["d2h_done"].record(st["d2h"])
            ev.record(st["d2h"])
        return _Pending(self, out, ev, err)

    def _pipeline(self):
        st = getattr(self, "_pipe", None)
        if st is None:
            t = _dev.torch()
            dev = self.w_gate.device
            h = max(self.tables.ngram_n, 1)
            if self.group is None:
                P = [self.partial, t.zeros_like(self.partial)]
                peer_P = [None, None]
            else:                              # both slots are peer-visible (IPC)
                P = [self._peer["partial_local"], self._peer["partial_b_local"]]
                peer_P = [self._peer["partial"], self._peer["partial_b"]]
            st = {"P": P, "peer_P": peer_P,
                  "tok": [t.zeros(self.max_tokens, dtype=t.int64, device=dev) for _ in range(2)],
                  "hist": [t.zeros((self.max_tokens, h), dtype=t.int64, device=dev)
                           for _ in range(2)],
                  "h2d": t.cuda.Stream(), "d2h": t.cuda.Stream(),
                  "compute": t.cuda.current_stream(),
                  "free_p": [t.cuda.Event(), t.cuda.Event()],
                  "free_ids": [t.cuda.Event(), t.cuda.Event()],
                  "in": [t.cuda.Event(), t.cuda.Event()],
                  "done": t.cuda.Event(), "d2h_done": t.cuda.Event(), "count": 0}
            for e in st["free_p"] + st["free_ids"] + [st["d2h_done"]]:
                e.record(st["compute"])
            self._pipe = st
        return st

    # ------------------------------------------------------------ results
    def check_errors(self):
        self._raise_for(int(self.err.item()))

    @staticmethod
    def _raise_for(bits: int):
        if bits & N.ERRBIT_TIMEOUT:
            raise RuntimeError("an in-kernel wait between the expert GEMMs timed out "
                               "(results invalid); SMOE_OPT_EARLY_DOWN = 0 disables it")
        if bits & N.ERRBIT_CAPACITY:
            raise SchedulerError("expert_rows capacity exceeded; raise expert_rows")
        if bits & N.ERRBIT_DEVICE_RANGE:
            raise SchedulerError("device label out of range")
        if bits & (N.ERRBIT_TOKEN_RANGE | N.ERRBIT_HISTORY_RANGE):
            raise IndexError("token id or history out of range")

    def plan_indices(self, n: int):
        """The ShuffleIndices of the last forward (bit-exact with
        scheduler.rebatch_tokens on the looked-up devices)."""
        from .scheduler import ShuffleIndices
        group = int(self.group_t.item())
        return ShuffleIndices(forward=self.forward_buf[: self.G * group].cpu().numpy(),
                              inverse=self.inverse[:n].cpu().numpy(), group_size=group,
                              n_devices=self.G)

    def routing(self, n: int):
        """Per original token: expert slots (s-EG order), ORIGINAL expert ids
        and weights, gathered from the shards' top-k buffers."""
        counts = self.plan_counts.cpu().numpy()
        group = int(self.group_t.item())
        fwd = self.forward_buf[: self.G * group].cpu().numpy()
        slots = np.full((n, self.k), -1, dtype=np.int64)
        wts = np.zeros((n, self.k), dtype=np.float32)
        ids = self.topk_ids.cpu().numpy()
        ws = self.topk_w.cpu().numpy()
        for i in range(self.shard_count):
            g = self.shard_begin + i
            c = int(counts[g])
            pos = fwd[g * group: g * group + c]
            slots[pos] = ids[i, :c]
            wts[pos] = ws[i, :c]
        experts = np.where(slots >= 0, np.asarray(self.perm.new_to_old)[np.maximum(slots, 0)], -1)
        return {"slots": slots, "experts": experts, "weights": wts}

    def stats(self, n: int | None = None) -> dict:
        """Locality and traffic of the last forward (mirrors the keys of
        comm.simulate_layer, comm.py:223-227, plus per-stage bytes)."""
        s = self.stats_t.cpu().numpy()
        local, remote = int(s[N.STAT_LOCAL_PAIRS]), int(s[N.STAT_REMOTE_PAIRS])
        counts = self.plan_counts.cpu().numpy().astype(np.int64)
        cm = self.counts_mat.cpu().numpy().astype(np.int64)
        group = int(self.group_t.item())
        n = int(counts.sum()) if n is None else n
        row = 2 * self.d
        G = self.G
        srs_bytes = int(counts.sum()) * (G - 1) * row      # rows pulled from other shards
        sag_bytes = int(counts.sum()) * (G - 1) * row      # rows pushed to other shards
        a2a = remote * row
        rrows = int(s[N.STAT_REMOTE_ROWS])
        # the dispatch sends one row per (token, remote shard) when the
        # deduplicated dispatch is on (SMOE_OPT_DEDUP_DISPATCH, the default),
        # else one per remote (token, expert) pair -- the reference's event
        # model (comm.py:86); the combine returns one row per remote pair
        dedup = bool(self.lib.smoe_get_option(N.OPT_DEDUP_DISPATCH))
        return {
            "local_tokens": local, "remote_tokens": remote,
            "measured_alpha": local / max(local + remote, 1),
            "group_size": group, "device_counts": counts.tolist(),
            "pair_counts": cm.tolist(),
            "bytes": {"srs": srs_bytes, "a2a_dispatch": (rrows if dedup else remote) * row,
                      "a2a_combine": a2a, "sag": sag_bytes,
                      "srs_padded_model": G * group * (G - 1) * row,
                      "reference_model_a2a": a2a,
                      "a2a_dispatch_dedup_model": rrows * row},
            "remote_rows": rrows,
            # rows the dispatch actually stored into other processes' shards
            # (deduplicated: one per (token, remote shard), SMOE_OPT_DEDUP_DISPATCH)
            "sent_rows": int(s[N.STAT_SENT_ROWS]),
        }


class _Pending:
    """Handle of a `forward_async` batch."""

    def __init__(self, layer, out, event, err):
        self._layer, self._out, self._event, self._err = layer, out, event, err

    def done(self) -> bool:
        return self._event.query()

    def result(self):
        # waits for this batch's D2H only: the compute stream keeps running
        # the next batch (a device-flag .item() here would drain it)
        self._event.synchronize()
        self._layer._raise_for(int(self._err[0]))
        return self._out


class MicroBatchedSpecMoE:
    """One MoE layer run as M micro-batches on M streams, so the HBM/NVLink
    stages of one micro-batch (SRS, gate, dispatch, combine+SAG) run while
    the persistent tcgen05 GEMMs of another occupy the tensor cores (the
    GEMM CTAs leave registers and shared memory for mover CTAs on every SM).

    Every token's result is independent of how the batch is cut, so the
    output is bit-identical to `SpecMoELayer`.  The micro-batch layers share
    the packed weights.  Single process: they write their partial inputs /
    outputs / next-layer histories through views of one full-size buffer (no
    copies).  With a ShardGroup each micro-batch layer has its own
    peer-visible (CUDA IPC) buffers and barrier epochs, every process builds
    the same micro-batches in the same order, and `forward` scatters the
    partials into them and gathers the outputs.

    On one GPU this is slower (the power cap); it exists for the
    multi-GPU case, where SRS / SAG are NVLink-bound and can overlap the
    power-bound GEMMs of the neighbouring micro-batch.
    """

    def __init__(self, bundle, gate_w, w1, w3, w2, *, top_k: int, max_tokens: int,
                 microbatches: int = 2, **kw):
        t = _dev.torch()
        self.group = kw.get("group")
        self.M = int(microbatches)
        self.max_tokens = int(max_tokens)
        self.chunk = -(-self.max_tokens // self.M)
        first = SpecMoELayer(bundle, gate_w, w1, w3, w2, top_k=top_k, max_tokens=self.chunk, **kw)
        self.layers = [first] + [
            SpecMoELayer(bundle, gate_w, None, None, None, top_k=top_k, max_tokens=self.chunk,
                         shared_from=first, **kw) for _ in range(self.M - 1)]
        G, d = first.G, first.d
        dev = first.w_gate.device
        self.G, self.d = G, d
        self.shard_count, self.shard_begin = first.shard_count, first.shard_begin
        self.streams = [t.cuda.current_stream()] + [t.cuda.Stream() for _ in range(self.M - 1)]
        self.events = [t.cuda.Event() for _ in range(self.M)]
        if self.group is not None:
            return                       # every micro-batch layer keeps its own IPC buffers
        self.partial = t.zeros((G, self.max_tokens, d), dtype=t.bfloat16, device=dev)
        self.out_buf = t.empty((self.max_tokens, d), dtype=t.bfloat16, device=dev)
        self.out = self.out_buf.unsqueeze(0).expand(G, self.max_tokens, d)
        h = max(first.tables.ngram_n, 1)
        self.hist_next = t.zeros((self.max_tokens, h), dtype=t.int64, device=dev)
        for c, L in enumerate(self.layers):
            lo = c * self.chunk
            hi = min(self.max_tokens, lo + self.chunk)
            P = self.partial[:, lo:hi]
            L._bind_partial(P)
            L.partial, L.out = P, self.out[:, lo:hi]       # drop the layer's own copies
            L.out_buf = self.out_buf[lo:hi]
            L._bound_partial = P
            for g in range(G):
                N.check(L.lib.smoe_layer_bind(L._h, N.BUF_OUT, g, N.ptr(self.out_buf[lo:])),
                        "bind")
                N.check(L.lib.smoe_layer_bind(L._h, N.BUF_HIST_OUT, g,
                                              N.ptr(self.hist_next[lo:])), "bind")

    def _pieces(self, n: int):
        out = []
        for c, L in enumerate(self.layers):
            lo = c * self.chunk
            hi = min(n, lo + self.chunk)
            if hi > lo:
                out.append((c, L, lo, hi))
        return out

    def partial_views(self, n: int):
        if self.group is not None:
            raise SchedulerError("with a ShardGroup each micro-batch has its own partial "
                                 "buffer: use forward() or load_partials()")
        return self.partial[:, :n]

    def load_partials(self, partials):
        """Copy this process's [L, n, d] partials into the micro-batch buffers."""
        n = int(partials.shape[1])
        for c, L, lo, hi in self._pieces(n):
            L.partial_views(hi - lo).copy_(partials[:, lo:hi], non_blocking=True)

    def out_view(self, n: int, shard: int = 0):
        if self.group is not None:
            t = _dev.torch()
            return t.cat([L.out_view(hi - lo) for c, L, lo, hi in self._pieces(n)])
        return self.out[shard, :n]

    def next_history(self, n: int):
        """As SpecMoELayer.next_history: None until the window is full."""
        win, depth = self.history_window(n)
        return win if depth >= self.layers[0].history_width and depth > 0 else None

    def history_window(self, n: int):
        depth = int(getattr(self.layers[0], "_hist_depth_out", 0))
        if self.group is not None:
            t = _dev.torch()
            return t.cat([L.history_window(hi - lo)[0] for c, L, lo, hi in self._pieces(n)]), depth
        return self.hist_next[:n], depth

    def forward(self, hidden_partials, token_ids, histories=None, history_depth=None):
        """[L, n, d] partials (device or host), token ids [n], histories
        [n, h]: the layer output [n, d] on the device."""
        t = _dev.torch()
        dev = self.layers[0].w_gate.device
        hp = t.as_tensor(hidden_partials)
        if hp.dim() == 2:
            hp = hp.unsqueeze(0)
        tok = t.as_tensor(token_ids).to(device=dev, dtype=t.int64).reshape(-1).contiguous()
        hist = None if histories is None else t.as_tensor(histories).to(
            device=dev, dtype=t.int64).contiguous()
        self.layers[0]._device_inputs(tok, hist, history_depth,   # validate the whole batch
                                      max_tokens=self.max_tokens)
        if self.group is None:
            self.partial_views(int(tok.numel())).copy_(hp)
        else:
            self.load_partials(hp.to(device=dev, dtype=t.bfloat16))
        out = self.run_device(tok, hist, history_depth)
        self.check_errors()
        return out

    def run_device(self, tokens_t, hist_t=None, hist_depth=None):
        """All micro-batches of one forward; returns the output view.  The
        GEMMs run in micro-batch order (each waits for the previous one's
        down projection), the movers of neighbouring micro-batches overlap
        them."""
        t = _dev.torch()
        n = int(tokens_t.shape[0])
        if n > self.max_tokens:
            raise SchedulerError(f"{n} tokens exceed max_tokens={self.max_tokens}")
        main = t.cuda.current_stream()
        for s in self.streams[1:]:
            s.wait_stream(main)
        pre = [N.STAGE_PLAN, N.STAGE_SRS, N.STAGE_GATE, N.STAGE_ROUTE, N.STAGE_DISPATCH]
        parts = self._pieces(n)
        for c, L, lo, hi in parts:                    # movers of every micro-batch first
            h = None if hist_t is None else hist_t[lo:hi]
            L.run_device(tokens_t[lo:hi], h, stream=self.streams[c], stages=pre,
                         hist_depth=hist_depth)
        prev = None
        for c, L, lo, hi in parts:                    # GEMMs in order, combine overlaps next
            s = self.streams[c]
            h = None if hist_t is None else hist_t[lo:hi]
            if prev is not None:
                s.wait_event(prev)
            L.run_device(tokens_t[lo:hi], h, stream=s,
                         stages=[N.STAGE_EXPERT_UP, N.STAGE_EXPERT_DOWN], hist_depth=hist_depth)
            self.events[c].record(s)
            prev = self.events[c]
            L.run_device(tokens_t[lo:hi], h, stream=s, stages=[N.STAGE_COMBINE_SAG],
                         hist_depth=hist_depth)
        for s in self.streams[1:]:
            main.wait_stream(s)
        return self.out_view(n)

    def check_errors(self):
        for L in self.layers:
            L.check_errors()

    def stats(self, n: int | None = None) -> dict:
        st = [L.stats() for L in self.layers]
        loc = sum(x["local_tokens"] for x in st)
        rem = sum(x["remote_tokens"] for x in st)
        return {"local_tokens": loc, "remote_tokens": rem,
                "measured_alpha": loc / max(loc + rem, 1),
                "bytes": {k: sum(x["bytes"][k] for x in st) for k in st[0]["bytes"]},
                "group_size": max(x["group_size"] for x in st),
                "microbatches": self.M}
