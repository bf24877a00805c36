"""BASELINE configs[4]: local-activation-rate sweep, s-MoE (SRS -> A2A -> A2A,
SAG) vs DS-MoE (AR -> A2A -> A2A -> AG), on skewed synthetic routing.

One GPU holds all G EP shards, so the collectives are HBM copies here; what
this measures per point is the routing (alpha), the bytes each stage moves
between shards (layer stats: what crosses NVLink when the G shards are G
GPUs), both pipelines' one-GPU step time (interleaved), and the projected
per-GPU NVLink time at G GPUs (per-GPU bytes / 770 GB/s measured peer-copy
rate, stages serial) next to the reference's volume model (comm.py).

    python tools/alpha_sweep.py [--configs mixtral:8,dsv2_lite:8,qwen2_57b:2,qwen2_57b:4,qwen2_57b:8]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

NVLINK_GBS = 770.0


def main():
    import torch
    from paper_2503_04398_b200 import SpecMoELayer, comm, synth
    from paper_2503_04398_b200.baseline import DSMoEPipelineLayer
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="mixtral:8,dsv2_lite:8,qwen2_57b:2,qwen2_57b:4,qwen2_57b:8")
    ap.add_argument("--eps", default="1.0,0.7,0.5,0.3,0.2,0.1,0.0")
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    n = a.tokens
    for spec in a.configs.split(","):
        name, G = spec.split(":")
        G = int(G)
        for eps in [float(x) for x in a.eps.split(",")]:
            cfg = dict(synth.CONFIGS[name])
            cfg["G"] = G
            w = synth.make_workload(name, n=n, eps=eps, seed=0, device=True, cfg_override=cfg)
            k, d = cfg["k"], cfg["d"]
            sm = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=k, max_tokens=n)
            sm.partial_views(n).copy_(w.partials)
            tok = torch.as_tensor(w.tokens, device="cuda")
            hist = torch.as_tensor(w.hist, device="cuda")
            ds = DSMoEPipelineLayer(w.gate_w, w.w1, w.w3, w.w2, n_ranks=G, top_k=k, max_tokens=n)
            ds.partial_views(n).copy_(w.partials)
            runs = {"smoe": lambda: sm.run_device(tok, hist), "dsmoe": lambda: ds.run_device(n=n)}
            ms = {"smoe": 0.0, "dsmoe": 0.0}
            for f in runs.values():
                f()
            torch.cuda.synchronize()
            for r in range(2):                                  # ABBA
                for key in (("smoe", "dsmoe") if r == 0 else ("dsmoe", "smoe")):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.steps):
                        runs[key]()
                    e1.record()
                    torch.cuda.synchronize()
                    ms[key] += e0.elapsed_time(e1) / (2 * a.steps)
            st, bt = sm.stats(n), ds.stats(n)
            b, bb = st["bytes"], bt["bytes"]
            per_gpu = lambda x: x / G                             # noqa: E731
            smoe_b = {"srs": b["srs"], "dispatch": b["a2a_dispatch"],
                      "dispatch_per_pair": b["reference_model_a2a"], "combine": b["a2a_combine"],
                      "sag": b["sag"]}
            ds_b = {"all_reduce": bb["all_reduce"], "dispatch": bb["a2a_dispatch"],
                    "combine": bb["a2a_combine"], "all_gather": bb["all_gather"]}
            s_tot = smoe_b["srs"] + smoe_b["dispatch"] + smoe_b["combine"] + smoe_b["sag"]
            s_tot_pp = s_tot - smoe_b["dispatch"] + smoe_b["dispatch_per_pair"]
            d_tot = sum(ds_b.values())
            alpha = st["measured_alpha"]
            model = comm.saving_ratio(comm.pipeline_volume(comm.dense_pipeline(G, 1, 1, k)),
                                      comm.pipeline_volume(comm.sharded_pipeline(G, 1, 1, k, alpha)))
            model_sag = comm.saving_ratio(
                comm.pipeline_volume(comm.dense_pipeline(G, 1, 1, k)),
                comm.pipeline_volume(comm.sharded_pipeline_with_sag(G, 1, 1, k, alpha)))
            print(json.dumps({
                "config": name, "G": G, "tokens": n, "eps": eps, "alpha": alpha,
                "alpha_dsmoe": bt["measured_alpha"],
                "smoe_bytes": smoe_b, "dsmoe_bytes": ds_b,
                "measured_saving": 1 - s_tot / d_tot,
                "measured_saving_per_pair_dispatch": 1 - s_tot_pp / d_tot,
                "model_saving": model, "model_saving_with_sag": model_sag,
                "projected_nvlink_ms_per_gpu": {
                    "smoe": per_gpu(s_tot) / (NVLINK_GBS * 1e6),
                    "dsmoe": per_gpu(d_tot) / (NVLINK_GBS * 1e6)},
                "one_gpu_ms": ms}), flush=True)
            del sm, ds, w
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
