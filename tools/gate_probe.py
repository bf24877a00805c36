"""Time the gate stage (K4) alone on the model configs, CUDA events, after a
full forward has produced the hidden rows.  Used for the tcgen05 gate's ring
shape (run once per SMOE_GATE_RING value: the choice is read once per process).

    SMOE_GATE_RING=2 python tools/gate_probe.py
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from paper_2503_04398_b200 import SpecMoELayer, _native as N, synth
    j = N.STAGE_NAMES.index("gate")
    for name, n, ep in (("mixtral", 16384, None), ("dsv2_lite", 16384, None),
                        ("dsv2_lite", 65536, None), ("qwen2_57b", 65536, 8)):
        over = {"G": ep} if ep else None
        w = synth.make_workload(name, n=n, eps=0.2, seed=0, device=True, cfg_override=over)
        layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"],
                             max_tokens=n)
        layer.partial_views(n).copy_(w.partials)
        d = w.cfg["d"]
        del w
        tok = torch.arange(n, device="cuda") % layer.tables.vocab
        layer.run_device(tok)
        torch.cuda.synchronize()
        for _ in range(3):
            layer.run_device(tok, stages=[j])
        reps = 50
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            layer.run_device(tok, stages=[j])
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        print(json.dumps({"config": name, "tokens": n, "ring": os.environ.get("SMOE_GATE_RING", "2"),
                          "gate_us": us, "gbs": n * d * 2 / us / 1e3}), flush=True)
        del layer
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
