"""Per-CTA timeline of the tcgen05 gate at decode sizes (needs the
instrumented probe build libsmoe_gateprobe.so via SMOE_LIB)."""
import ctypes as C
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
j = N.STAGE_NAMES.index("gate")
layer.run_device(tok, hist, stages=[0, 1])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); layer.run_device(tok, hist, stages=[j]); e1.record(); torch.cuda.synchronize()
h = N.load()
buf = (C.c_ulonglong * (512 * 8))()
fn = getattr(h, "smoe_probe_gate_ts"); fn.restype = C.c_int
assert fn(buf, 512) == 0
ts = np.frombuffer(buf, dtype=np.uint64).reshape(512, 8).astype(np.int64)
act = ts[(ts[:, 4] > 0) & (ts[:, 0] > 0)]
base = ts[ts[:, 0] > 0, 0].min()
print(f"{name} n={n}: event {e0.elapsed_time(e1)*1e3:.1f} us, CTAs with a tile {len(act)}")
for r in act[:4]:
    print("  start+%.1f setup %.1f  producer_done %.1f  mma_done %.1f  tfull_seen %.1f  epi_done %.1f  exit %.1f (us from CTA start)"
          % ((r[0]-base)/1e3, (r[1]-r[0])/1e3, (r[2]-r[0])/1e3, (r[3]-r[0])/1e3, (r[4]-r[0])/1e3, (r[5]-r[0])/1e3, (r[6]-r[0])/1e3))
