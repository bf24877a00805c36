"""Worker bodies for the multi-process tests (spawned; module-level for pickling)."""

import os

import numpy as np


def layer_worker(rank, world, port, cfg_over, n, result_q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)                      # every rank on one GPU (IPC still applies)
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
