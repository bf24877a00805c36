"""Shards spread over processes: peer buffers over CUDA IPC (NVLink P2P).

One process per GPU, `torch.distributed` for the plumbing only: the IPC
handles of every process's peer-visible buffers are exchanged once with
`all_gather_object`; after that the layer's kernels read and write peer HBM
directly (SRS pulls partial rows, dispatch / the down-GEMM epilogue / SAG
push rows) and synchronise through signal pads (smoe_layer_barrier).  No
NCCL call sits on the s-MoE data path.

Process r owns shards [r*L, (r+1)*L), L = G / world_size.
"""

from __future__ import annotations

import ctypes as C

from . import _native as N


class _CudaArray:
    """__cuda_array_interface__ view of a raw device allocation (for torch.as_tensor)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3, "strides": None}


class ShardGroup:
    def __init__(self, world_size: int, rank: int, allgather):
        """allgather(obj) -> list of obj from every rank (rank order)."""
        self.world_size = int(world_size)
        self.rank = int(rank)
        self._allgather = allgather
        self._owned: list[int] = []
        self._opened: list[int] = []

    @classmethod
    def from_torch_distributed(cls, group=None):
        import torch.distributed as dist
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)

        def allgather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj, group=group)
            return out
        return cls(world, rank, allgather)

    # ------------------------------------------------------------------ memory
    def _alloc(self, nbytes: int) -> int:
        lib = N.lib()
        p = C.c_void_p()
        N.check(lib.smoe_device_alloc(max(int(nbytes), 256), C.byref(p)), "device_alloc")
        self._owned.append(p.value)
        return int(p.value)

    def _ipc_handle(self, ptr: int) -> bytes:
        h = (C.c_char * 64)()
        N.check(N.lib().smoe_ipc_handle(ptr, h), "ipc_handle")
        return bytes(h)

    def _ipc_open(self, handle: bytes) -> int:
        out = C.c_void_p()
        buf = (C.c_char * 64).from_buffer_copy(handle)
        N.check(N.lib().smoe_ipc_open(buf, C.byref(out)), "ipc_open")
        self._opened.append(int(out.value))
        return int(out.value)

    def _exchange(self, ptr: int) -> list[int]:
        """Every rank's base pointer of one allocation, mapped into this process."""
        handles = self._allgather(self._ipc_handle(ptr))
        return [ptr if r == self.rank else self._ipc_open(hb) for r, hb in enumerate(handles)]

    def peer_tables(self, G: int, n_experts: int, per_shard: dict,
                    per_process: dict | None = None) -> tuple[dict, dict]:
        """Allocate this process's share of every peer buffer and build the
        per-shard pointer tables (shard g lives on process g // L at offset
        (g % L) * size).  Returns (tables, local base pointers)."""
        L = G // self.world_size
        peer, local = {}, {}
        for name, size in per_shard.items():
            base = self._alloc(size * L)
            bases = self._exchange(base)
            peer[name] = [bases[g // L] + (g % L) * size for g in range(G)]
            local[name] = base
        procs = {"counts": G * n_experts * 4, "signal": 64 * 4, **(per_process or {})}
        for name, size in procs.items():
            base = self._alloc(size)
            bases = self._exchange(base)
            peer[name] = [bases[g // L] for g in range(G)]
            local[name] = base
        return peer, local

    def alloc_layer_buffers(self, layer, device):
        import torch
        G, L = layer.G, layer.shard_count
        n, d, k, R = layer.max_tokens, layer.d, layer.k, layer.expert_rows
        # two partial-input buffers: forward_async fills one while the peers'
        # SRS reads the other
        per_shard = {"partial": n * d * 2, "partial_b": n * d * 2, "xin": R * d * 2,
                     "xmeta": R * 8, "xfan": R * 4, "ypair": n * k * d * 2}
        h = max(int(layer.tables.ngram_n), 1)
        # one output (and next-layer history) per process: the SAG delivers
        # every token's row to each process once, whichever of its shards
        extra = layer.process_row_buffers()      # e.g. the DS-MoE pipeline's AR / AG
        peer, local = self.peer_tables(G, layer.N, per_shard,
                                       {"hist": n * h * 8, "out": n * d * 2,
                                        **{name: rows * d * 2 for name, rows in extra.items()}})

        def tensor(ptr, shape, typestr):
            return torch.as_tensor(_CudaArray(ptr, shape, typestr), device=device)

        # bf16 has no array-interface typestr: view int16 storage as bfloat16
        peer["partial_local"] = tensor(local["partial"], (L, n, d), "<i2").view(torch.bfloat16)
        peer["partial_b_local"] = tensor(local["partial_b"], (L, n, d),
                                         "<i2").view(torch.bfloat16)
        peer["out_local"] = tensor(local["out"], (n, d), "<i2").view(torch.bfloat16)
        peer["xin_local"] = tensor(local["xin"], (L, R, d), "<i2").view(torch.bfloat16)
        for name, rows in extra.items():
            peer[name + "_local"] = tensor(local[name], (rows, d), "<i2").view(torch.bfloat16)
        peer["counts_local"] = tensor(local["counts"], (G, layer.N), "<i4")
        peer["hist_local"] = tensor(local["hist"], (n, h), "<i8")
        tensor(local["signal"], (64,), "<i4").zero_()
        peer["partial_local"].zero_()
        peer["partial_b_local"].zero_()
        torch.cuda.synchronize()
        self._allgather(0)                 # every pad is zero before anyone signals
        return peer

    def close(self):
        lib = N.load()
        for p in self._opened:
            lib.smoe_ipc_close(p)
        for p in self._owned:
            lib.smoe_device_free(p)
        self._opened.clear()
        self._owned.clear()
