"""A2A bytes per forward: per (token, expert) pair (the reference model, what
the dispatch sends) vs one row per (token, destination shard)."""
import json
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import SpecMoELayer, synth
for name in ("mixtral", "dsv2_lite", "qwen2_57b"):
    for eps in (0.0, 0.2, 0.5):
        n = 16384
        w = synth.make_workload(name, n=n, eps=eps, seed=0, device=True)
        layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"], max_tokens=n)
        layer.partial_views(n).copy_(w.partials)
        layer.run_device(torch.as_tensor(w.tokens, device="cuda"), torch.as_tensor(w.hist, device="cuda"))
        torch.cuda.synchronize()
        st = layer.stats(n)
        b = st["bytes"]
        print(json.dumps({"config": name, "eps": eps, "alpha": st["measured_alpha"],
                          "a2a_dispatch_bytes": b["a2a_dispatch"],
                          "dedup_bytes": b["a2a_dispatch_dedup_model"],
                          "dedup_ratio": b["a2a_dispatch_dedup_model"] / max(b["a2a_dispatch"], 1)}),
              flush=True)
        del layer, w
        torch.cuda.empty_cache()
