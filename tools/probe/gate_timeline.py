"""Per-CTA timeline of the tcgen05 gate (instrumented build):

    python -m paper_2503_04398_b200.build --variant gateprobe -DSMOE_GATE_PROBE
    SMOE_LIB=$PWD/paper_2503_04398_b200/libsmoe_gateprobe.so python tools/probe/gate_timeline.py dsv2_lite 16384

Points (per CTA, first tile, %globaltimer ns): 0 entry, 1 set-up done (TMEM,
barriers, counts), 2 last TMA of the tile issued, 3 first stage landed, 4 last
MMA issued, 5 accumulator ready in the epilogue, 6 epilogue warp done, 7 exit;
register epilogue (first thread): 8 logits in registers, 9 k selections done,
10 softmax sum + exchange written, 11 halves merged, 12 stats atomics done,
14 fused route done.
Prints the median / max over CTAs of each point relative to the earliest entry.
"""
import ctypes as C
import json
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
from paper_2503_04398_b200 import SpecMoELayer, synth, _native as N
name, n = sys.argv[1], int(sys.argv[2])
w = synth.make_workload(name, n=n, eps=0.2, seed=0, device=True)
layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=w.cfg["k"], max_tokens=n)
layer.partial_views(n).copy_(w.partials)
tok = torch.as_tensor(w.tokens, device="cuda"); hist = torch.as_tensor(w.hist, device="cuda")
for _ in range(3):
    layer.run_device(tok, hist)
torch.cuda.synchronize()
h = N.lib()
j = N.STAGE_NAMES.index("gate")
junk = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
out = []
for rep in range(3):
    layer.run_device(tok, hist, stages=[0, 1])
    junk.fill_(rep)                                   # cold L2, like the layer after the SRS
    torch.cuda.synchronize()
    assert h.smoe_probe_gate_reset() == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); layer.run_device(tok, hist, stages=[j]); e1.record(); torch.cuda.synchronize()
    buf = (C.c_ulonglong * (2048 * 16))()
    assert h.smoe_probe_gate_ts(buf, 2048) == 0
    ts = np.frombuffer(buf, dtype=np.uint64).reshape(2048, 16).astype(np.int64)
    act = ts[(ts[:, 0] > 0) & (ts[:, 5] > 0)]
    base = ts[ts[:, 0] > 0, 0].min()
    rel = (act - base) / 1e3
    out.append({"config": name, "tokens": n, "event_us": e0.elapsed_time(e1) * 1e3,
                "ctas_with_tile": int(len(act)),
                "median_us": [round(float(x), 2) for x in np.median(rel, axis=0)],
                "max_us": [round(float(x), 2) for x in rel.max(axis=0)]})
    print(json.dumps(out[-1]), flush=True)
