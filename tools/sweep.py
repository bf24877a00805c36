"""Config x tokens x skew sweep of the MoE layer on one GPU (EP shards
emulated on the device), BASELINE.json configs[1..4].  One JSON line per
point; used for profiles/r*_sweep.jsonl.

    python tools/sweep.py [--quick]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def measure(name, tokens, eps, ep=None, steps=10, warmup=3, seed=0, microbatches=1):
    import torch
    from paper_2503_04398_b200 import SpecMoELayer, comm, synth
    from paper_2503_04398_b200 import _native as N
    cfg = dict(synth.CONFIGS[name])
    if ep:
        cfg["G"] = ep
    G, k, d, f = cfg["G"], cfg["k"], cfg["d"], cfg["f"]
    t0 = time.time()
    w = synth.make_workload(name, n=tokens, eps=eps, seed=seed, device=True, cfg_override=cfg)
    if microbatches > 1:
        from paper_2503_04398_b200.layer import MicroBatchedSpecMoE
        layer = MicroBatchedSpecMoE(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=k,
                                    max_tokens=tokens, microbatches=microbatches)
    else:
        layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=k, max_tokens=tokens)
    layer.partial_views(tokens).copy_(w.partials)
    del w.partials
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    for _ in range(warmup):
        layer.run_device(tok, hist)
    torch.cuda.synchronize()
    layer.check_errors()
    if microbatches > 1:
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(steps):
            layer.run_device(tok, hist)
        e1.record(s)
        torch.cuda.synchronize()
        step_ms = e0.elapsed_time(e1) / steps
        st = layer.stats(tokens)
        out = {"config": name, "ep": G, "tokens": tokens, "eps": eps, "microbatches": microbatches,
               "alpha": st["measured_alpha"], "ms_per_step": step_ms,
               "tokens_per_s": tokens / (step_ms / 1e3), "setup_s": time.time() - t0}
        del layer
        torch.cuda.empty_cache()
        return out
    names = N.STAGE_NAMES
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
          for _ in range(steps)]
    s = torch.cuda.current_stream()
    for i in range(steps):
        ev[i][0].record(s)
        for j in range(len(names)):
            layer.run_device(tok, hist, stages=[j])
            ev[i][j + 1].record(s)
    torch.cuda.synchronize()
    stage_ms = {nm: float(np.mean([ev[i][j].elapsed_time(ev[i][j + 1]) for i in range(steps)]))
                for j, nm in enumerate(names)}
    step_ms = float(np.mean([ev[i][0].elapsed_time(ev[i][-1]) for i in range(steps)]))
    st = layer.stats(tokens)
    pairs = st["local_tokens"] + st["remote_tokens"]
    a = st["measured_alpha"]
    dense = comm.pipeline_volume(comm.dense_pipeline(G, 1, tokens, k)).total
    model = comm.pipeline_volume(comm.sharded_pipeline(G, 1, tokens, k, a)).total
    sag = comm.pipeline_volume(comm.sharded_pipeline_with_sag(G, 1, tokens, k, a)).total
    flops = 6.0 * pairs * d * f
    out = {"config": name, "ep": G, "tokens": tokens, "eps": eps, "alpha": a,
           "group": st["group_size"], "ms_per_step": step_ms,
           "tokens_per_s": tokens / (step_ms / 1e3),
           "expert_tflops": flops / ((stage_ms["expert_up"] + stage_ms["expert_down"]) / 1e3) / 1e12,
           "stage_ms": stage_ms, "a2a_bytes": st["bytes"]["a2a_dispatch"] * 2,
           "predicted_saving_vs_dsmoe": {"model": 1 - model / dense, "with_sag": 1 - sag / dense},
           "setup_s": time.time() - t0}
    del layer
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--microbatch-ab", action="store_true",
                    help="interleaved 1 vs 2 vs 4 micro-batches on the main configs")
    ap.add_argument("--gate-ab", action="store_true",
                    help="interleaved tcgen05 gate vs mma.sync gate (SMOE_OPT_GATE_TENSOR)")
    ap.add_argument("--batch-sweep", action="store_true",
                    help="configs x 64 ... 65536 tokens (the DESIGN batch table)")
    args = ap.parse_args()
    if args.batch_sweep:
        for name, ep in (("mixtral", None), ("dsv2_lite", None), ("qwen2_57b", 8)):
            for tok in (64, 512, 2048, 8192, 16384, 65536):
                print(json.dumps(measure(name, tok, 0.2, ep)), flush=True)
        for ep in (4, 2):
            for tok in (2048, 16384):
                print(json.dumps(measure("qwen2_57b", tok, 0.2, ep)), flush=True)
        return
    if args.gate_ab:
        from paper_2503_04398_b200 import _native as N
        lib = N.lib()
        for rep in range(2):
            for name, tok, ep in (("mixtral", 16384, None), ("dsv2_lite", 16384, None),
                                  ("dsv2_lite", 65536, None), ("qwen2_57b", 65536, 8)):
                for opt in (1, 0):
                    N.check(lib.smoe_set_option(N.OPT_GATE_TENSOR, opt), "opt")
                    r = measure(name, tok, 0.2, ep)
                    print(json.dumps({k: r[k] for k in ("config", "tokens", "ms_per_step",
                                                        "tokens_per_s", "alpha")} |
                                     {"gate_ms": r["stage_ms"]["gate"], "gate_tensor": opt,
                                      "rep": rep}), flush=True)
        N.check(lib.smoe_set_option(N.OPT_GATE_TENSOR, 1), "opt")
        return
    if args.microbatch_ab:
        for rep in range(2):
            for name, tok in (("mixtral", 16384), ("dsv2_lite", 16384), ("qwen2_57b", 16384),
                              ("mixtral", 65536)):
                for mb in (1, 2, 4):
                    r = measure(name, tok, 0.2, microbatches=mb)
                    print(json.dumps({k: r[k] for k in ("config", "tokens", "ms_per_step",
                                                        "tokens_per_s", "alpha")} |
                                     {"microbatches": mb, "rep": rep}), flush=True)
        return
    pts = [("mixtral", 4096, 0.2, None), ("mixtral", 16384, 0.2, None),
           ("mixtral", 65536, 0.2, None),
           ("dsv2_lite", 16384, 0.2, None), ("dsv2_lite", 65536, 0.2, None),
           ("qwen2_57b", 16384, 0.2, 2), ("qwen2_57b", 16384, 0.2, 4),
           ("qwen2_57b", 16384, 0.2, 8), ("qwen2_57b", 65536, 0.2, 8)]
    for e in (0.0, 0.25, 0.5, 0.75, 1.0):
        pts.append(("dsv2_lite", 16384, e, None))
        pts.append(("mixtral", 16384, e, None))
    if args.quick:
        pts = pts[:2]
    for p in pts:
        print(json.dumps(measure(*p)), flush=True)


if __name__ == "__main__":
    main()
