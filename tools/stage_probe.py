"""Time single layer stages alone on the model configs, CUDA events, after a
full forward has produced every stage's inputs.  Used for kernel tuning knobs
that are read once per process (SMOE_GATE_RING, SMOE_SRS_U, ...):

    SMOE_GATE_RING=2 python tools/stage_probe.py --stages gate
    SMOE_SRS_U=1 python tools/stage_probe.py --stages plan,srs,combine_sag
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import argparse
    import torch
    from paper_2503_04398_b200 import SpecMoELayer, _native as N, synth
    ap = argparse.ArgumentParser()
    ap.add_argument("--stages", default="gate")
    ap.add_argument("--tokens", type=int, default=0, help="override every config's token count")
    ap.add_argument("--flush", action="store_true",
                    help="write 512 MiB before every timed call (cold L2) and time each call")
    args = ap.parse_args()
    knobs = {k: v for k, v in os.environ.items() if k.startswith("SMOE_")}
    cfgs = (("mixtral", 16384, None), ("dsv2_lite", 16384, None),
            ("dsv2_lite", 65536, None), ("qwen2_57b", 65536, 8), ("deepseek_v2", 16384, None))
    only = os.environ.get("SMOE_PROBE_CFGS")          # comma list of config names
    for name, n, ep in cfgs:
        if (only and name not in only.split(",")) or (not only and name == "deepseek_v2"):
            continue
        if args.tokens:
            if n == 65536 and name == "dsv2_lite":
                continue
            n = args.tokens
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
        for st in args.stages.split(","):
            j = N.STAGE_NAMES.index(st)
            for _ in range(3):
                layer.run_device(tok, stages=[j])
            reps = 50
            if args.flush:
                junk = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(reps)]
                for a, b in evs:
                    junk.fill_(1)
                    a.record()
                    layer.run_device(tok, stages=[j])
                    b.record()
                torch.cuda.synchronize()
                us = sum(a.elapsed_time(b) for a, b in evs) / reps * 1e3
                del junk
            else:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(reps):
                    layer.run_device(tok, stages=[j])
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / reps * 1e3
            print(json.dumps({"config": name, "tokens": n, "stage": st, "us": us,
                              "cold_l2": bool(args.flush),
                              "hidden_row_gbs": n * d * 2 / us / 1e3} | knobs), flush=True)
        del layer
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
