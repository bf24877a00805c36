"""A/B of SpecMoELayer vs MicroBatchedSpecMoE (M micro-batches on their own
streams) on N GPUs — the overlap of NVLink-bound SRS / SAG with the
power-bound GEMMs only pays when shards span GPUs.

    python tools/microbatch_bench.py --config mixtral --tokens 16384 --mb 2
    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \
        tools/microbatch_bench.py --mb 2

Interleaved reps, CUDA events, max over ranks; rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--tokens", type=int, default=16384, help="tokens per GPU")
    ap.add_argument("--mb", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    from paper_2503_04398_b200 import SpecMoELayer, synth
    from paper_2503_04398_b200.layer import MicroBatchedSpecMoE
    group = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2503_04398_b200.dist import ShardGroup
        group = ShardGroup.from_torch_distributed()
    n = a.tokens * world
    w = synth.make_workload(a.config, n=n, eps=0.2, seed=0, device=True)
    plain = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"], max_tokens=n,
                         group=group)
    mb = MicroBatchedSpecMoE(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"],
                             max_tokens=n, microbatches=a.mb, group=group)
    L, b0 = plain.shard_count, plain.shard_begin
    mine = w.partials[b0:b0 + L]
    plain.partial_views(n).copy_(mine)
    if group is None:
        mb.partial_views(n).copy_(mine)
    else:
        mb.load_partials(mine)
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")

    def timed(layer):
        for _ in range(2):
            layer.run_device(tok, hist)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            layer.run_device(tok, hist)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    res = {"plain": [], "microbatched": []}
    for _ in range(a.reps):
        res["plain"].append(timed(plain))
        res["microbatched"].append(timed(mb))
    if int(os.environ.get("RANK", "0")) == 0:
        best = {k: min(v) for k, v in res.items()}
        print(json.dumps({"config": a.config, "n_gpus": world, "tokens_per_gpu": a.tokens,
                          "microbatches": a.mb, "ms_per_step": best,
                          "tokens_per_s": {k: n / (v / 1e3) for k, v in best.items()},
                          "reps_ms": res}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
