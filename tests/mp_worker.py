"""Worker bodies for the multi-process tests (spawned; module-level for pickling)."""

import os

import numpy as np


def collect(q, procs, timeout=540):
    """One result per process from `q`, keyed by rank (the first tuple item).
    Fails fast when a worker dies instead of waiting out the timeout."""
    import queue
    import time
    res = {}
    deadline = time.monotonic() + timeout
    while len(res) < len(procs):
        try:
            item = q.get(timeout=5)
            res[item[0]] = item[1:]
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if dead or time.monotonic() > deadline:
                for p in procs:
                    p.kill()
                raise RuntimeError(f"worker failed (exit codes {dead}) or timed out")
    for p in procs:
        p.join(timeout=60)
        if p.exitcode != 0:
            raise RuntimeError(f"worker exit code {p.exitcode}")
    return res


def bind_device(rank, world):
    """Rank r on cuda:r when the box has a GPU per rank (then the IPC peer
    buffers, peer stores and signal-pad barriers really cross NVLink);
    otherwise every rank on cuda:0 (IPC within one GPU)."""
    import torch
    dev = rank if torch.cuda.device_count() >= world else 0
    torch.cuda.set_device(dev)
    return dev


def layer_worker(rank, world, port, cfg_over, n, result_q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    bind_device(rank, world)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_04398_b200 import SpecMoELayer, synth
        from paper_2503_04398_b200.dist import ShardGroup
        w = synth.make_workload("toy", n=n, eps=0.3, seed=11, cfg_override=cfg_over)
        grp = ShardGroup.from_torch_distributed()
        layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"],
                             max_tokens=n, group=grp)
        L = layer.shard_count
        mine = torch.from_numpy(w.partials[layer.shard_begin:layer.shard_begin + L])
        outs = []
        for _ in range(2):                          # twice: barrier epochs advance
            out = layer.forward(mine.cuda(), w.tokens, w.hist)
            outs.append(out.float().cpu().numpy())
        st = layer.stats_t.cpu().numpy()[:2].tolist()
        all_out = [layer.out[i, :n].float().cpu().numpy() for i in range(L)]
        result_q.put((rank, outs, st, all_out))
        dist.barrier()
        grp.close()
    finally:
        dist.destroy_process_group()


def async_worker(rank, world, port, cfg_over, sizes, result_q):
    """forward_async over several batches with FRESH partials each (every
    process writes its slot while peers may still read the other one)."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    bind_device(rank, world)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_04398_b200 import SpecMoELayer, synth
        from paper_2503_04398_b200.dist import ShardGroup
        ws = [synth.make_workload("toy", n=n, eps=0.3, seed=20 + i, cfg_override=cfg_over)
              for i, n in enumerate(sizes)]
        base = ws[0]
        grp = ShardGroup.from_torch_distributed()
        layer = SpecMoELayer(base.bundle, base.gate_w, base.w1, base.w3, base.w2,
                             top_k=base.cfg["k"], max_tokens=max(sizes), group=grp)
        L, b0 = layer.shard_count, layer.shard_begin
        pins = [(torch.from_numpy(w.partials[b0:b0 + L]).to(torch.bfloat16).pin_memory(),
                 torch.from_numpy(w.tokens).pin_memory(), torch.from_numpy(w.hist).pin_memory())
                for w in ws]
        outs = [torch.empty((len(w.tokens), base.cfg["d"]), dtype=torch.bfloat16).pin_memory()
                for w in ws]
        handles = [layer.forward_async(p, t, h, out=outs[i]) for i, (p, t, h) in enumerate(pins)]
        got = [hd.result().float().numpy() for hd in handles]
        result_q.put((rank, got))
        dist.barrier()
        grp.close()
    finally:
        dist.destroy_process_group()


def capture_worker(rank, world, port, cfg_over, seeds, n, result_q):
    """CUDA-graph capture of a multi-process layer; replays with new partials."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    bind_device(rank, world)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_04398_b200 import SpecMoELayer, synth
        from paper_2503_04398_b200.dist import ShardGroup
        ws = [synth.make_workload("toy", n=n, eps=0.3, seed=s, cfg_override=cfg_over) for s in seeds]
        base = ws[0]
        grp = ShardGroup.from_torch_distributed()
        layer = SpecMoELayer(base.bundle, base.gate_w, base.w1, base.w3, base.w2,
                             top_k=base.cfg["k"], max_tokens=n, group=grp)
        L, b0 = layer.shard_count, layer.shard_begin
        tok = torch.as_tensor(base.tokens, device="cuda")
        hist = torch.as_tensor(base.hist, device="cuda")
        layer.partial_views(n).copy_(torch.from_numpy(base.partials[b0:b0 + L]))
        g = layer.capture(tok, hist)
        got = []
        for w in ws:
            layer.partial_views(n).copy_(torch.from_numpy(w.partials[b0:b0 + L]))
            g.replay()
            torch.cuda.synchronize()
            layer.check_errors()
            got.append(layer.out_view(n).float().cpu().numpy())
        result_q.put((rank, got))
        dist.barrier()
        grp.close()
    finally:
        dist.destroy_process_group()


def microbatch_worker(rank, world, port, cfg_over, n, M, result_q):
    """MicroBatchedSpecMoE across processes: per-micro-batch IPC buffers."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    bind_device(rank, world)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_04398_b200 import synth
        from paper_2503_04398_b200.dist import ShardGroup
        from paper_2503_04398_b200.layer import MicroBatchedSpecMoE
        w = synth.make_workload("toy", n=n, eps=0.3, seed=12, cfg_override=cfg_over)
        grp = ShardGroup.from_torch_distributed()
        layer = MicroBatchedSpecMoE(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"],
                                    max_tokens=n, microbatches=M, group=grp)
        L, b0 = layer.shard_count, layer.shard_begin
        mine = torch.from_numpy(w.partials[b0:b0 + L])
        outs = []
        for _ in range(2):
            outs.append(layer.forward(mine, w.tokens, w.hist).float().cpu().numpy())
        hist = layer.next_history(n).cpu().numpy()
        result_q.put((rank, outs, hist))
        dist.barrier()
        grp.close()
    finally:
        dist.destroy_process_group()


def dsmoe_worker(rank, world, port, cfg_over, n, backend, result_q):
    """DSMoELayer(distributed=True): one DS-MoE rank per process.  NCCL when
    every rank has its own GPU; gloo (collectives staged through host
    memory) when the ranks share one GPU."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = bind_device(rank, world)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_04398_b200 import synth
        from paper_2503_04398_b200.baseline import DSMoELayer
        w = synth.make_workload("toy", n=n, eps=0.3, seed=5, cfg_override=cfg_over)
        layer = DSMoELayer(w.gate_w, w.w1, w.w3, w.w2, n_ranks=world, top_k=w.cfg["k"],
                           max_tokens=n, distributed=True)
        mine = torch.from_numpy(w.partials[rank]).to(torch.bfloat16).cuda()
        outs = [layer.forward([mine], n).float().cpu().numpy() for _ in range(2)]
        st = layer.stats()
        result_q.put((rank, outs, (st["local_tokens"], st["remote_tokens"])))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def dsmoe_pipeline_worker(rank, world, port, cfg_over, n, result_q):
    """DSMoEPipelineLayer over a ShardGroup: G / world shards per process."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    bind_device(rank, world)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_04398_b200 import synth
        from paper_2503_04398_b200.baseline import DSMoEPipelineLayer
        from paper_2503_04398_b200.dist import ShardGroup
        w = synth.make_workload("toy", n=n, eps=0.3, seed=12, cfg_override=cfg_over)
        grp = ShardGroup.from_torch_distributed()
        layer = DSMoEPipelineLayer(w.gate_w, w.w1, w.w3, w.w2, n_ranks=w.cfg["G"],
                                   top_k=w.cfg["k"], max_tokens=n, group=grp)
        L = layer.shard_count
        mine = torch.from_numpy(w.partials[layer.shard_begin:layer.shard_begin + L]).cuda()
        outs = [layer.forward(mine).float().cpu().numpy() for _ in range(2)]
        st = layer.stats_t.cpu().numpy()[:2].tolist()
        result_q.put((rank, outs, tuple(int(x) for x in st)))
        dist.barrier()
        grp.close()
    finally:
        dist.destroy_process_group()


def dedup_worker(rank, world, port, cfg_over, n, dedup, result_q):
    """SpecMoELayer over a ShardGroup with the deduplicated dispatch on / off:
    outputs and the rows the dispatch stored into other processes."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    bind_device(rank, world)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_04398_b200 import SpecMoELayer, synth, _native as N
        from paper_2503_04398_b200.dist import ShardGroup
        N.check(N.lib().smoe_set_option(N.OPT_DEDUP_DISPATCH, int(dedup)), "set_option")
        w = synth.make_workload("toy", n=n, eps=0.3, seed=21, cfg_override=cfg_over)
        grp = ShardGroup.from_torch_distributed()
        layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"],
                             max_tokens=n, group=grp)
        L = layer.shard_count
        mine = torch.from_numpy(w.partials[layer.shard_begin:layer.shard_begin + L]).cuda()
        outs = [layer.forward(mine, w.tokens, w.hist).float().cpu().numpy() for _ in range(2)]
        result_q.put((rank, outs, layer.stats()["sent_rows"]))
        dist.barrier()
        grp.close()
    finally:
        dist.destroy_process_group()
