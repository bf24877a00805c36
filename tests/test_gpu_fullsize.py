"""The layer at BASELINE.json's full sizes (configs[1..3]: Mixtral-8x7B,
DeepSeek-V2-Lite, Qwen2-57B-A14B layers, 16 384 tokens, EP 8) checked through
size-independent properties, since the CPU oracle would take minutes here:

* plan: counts sum to n, group = max count, forward/inverse are inverse
  permutations, pads are -1, every group keeps token order (stability), and
  the looked-up devices equal the reference lookup (oracle, numpy) bit-exactly;
* routing: the ordered top-k experts equal the planted choice (synth builds
  margin-guarded logits), local + remote = n*k, local = #{label(expert) = device};
* output: every token against a torch fp32 restatement of the layer (SRS
  sum in shard order -> bf16, fp32 gate softmax, fp32 SwiGLU on the bf16
  weights, renormalised top-k combine); relative Frobenius error <= 1e-2,
  every row <= 2e-2 (row norm), every element <= 2e-2 of its row's peak;
* next-layer history: shifted window + cluster of the top-1 expert.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import scheduler_ref as S
from paper_2503_04398_b200 import SpecMoELayer, synth

TOL = 1e-2


@pytest.mark.parametrize("name,ep", [("mixtral", 8), ("dsv2_lite", 8), ("qwen2_57b", 8),
                                     ("qwen2_57b", 2), ("deepseek_v2", 8)])
def test_full_size_layer_properties(name, ep):
    n = 16384
    w = synth.make_workload(name, n=n, eps=0.2, seed=3, device=True, cfg_override={"G": ep})
    G, k, d = w.cfg["G"], w.cfg["k"], w.cfg["d"]
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=k, max_tokens=n)
    layer.partial_views(n).copy_(w.partials)
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    out = layer.run_device(tok, hist).clone()
    torch.cuda.synchronize()
    layer.check_errors()

    # ---- plan
    tab = w.bundle
    dev_ref = S.lookup_devices(tab.token_table.labels, tab.token_table.confidence,
                               tab.ngram_table.best, tab.ngram_table.confidence, G, w.tokens,
                               w.hist)
    assert np.array_equal(layer.dev[:n].cpu().numpy(), dev_ref)
    ix = layer.plan_indices(n)
    counts = layer.plan_counts.cpu().numpy()
    assert counts.sum() == n and ix.group_size == counts.max()
    assert np.array_equal(counts, np.bincount(dev_ref, minlength=G))
    assert np.array_equal(ix.forward[ix.inverse], np.arange(n))
    for g in range(G):
        seg = ix.forward[g * ix.group_size:(g + 1) * ix.group_size]
        real = seg[: counts[g]]
        assert np.all(seg[counts[g]:] == -1)
        assert np.all(np.diff(real) > 0)                   # stable
        assert np.all(dev_ref[real] == g)

    # ---- routing and event counts
    r = layer.routing(n)
    assert np.array_equal(r["experts"], w.chosen)
    st = layer.stats()
    labels = np.asarray(w.expert_labels)
    local = int(np.count_nonzero(labels[w.chosen] == dev_ref[:, None]))
    assert st["local_tokens"] == local and st["remote_tokens"] == n * k - local

    # ---- next-layer history
    hn = layer.next_history(n).cpu().numpy()
    assert np.array_equal(hn[:, -1], labels[w.chosen[:, 0]])
    assert np.array_equal(hn[:, :-1], w.hist[:, 1:])

    # ---- output vs a torch fp32 restatement on EVERY token (the fp32
    # reference of the whole batch is a few TFLOP: well under a second here)
    sample = torch.arange(n, device="cuda")
    P = w.partials[:, sample].float()                      # [G, s, d]
    h = P[0].clone()
    for g in range(1, G):
        h = h + P[g]
    h = h.to(torch.bfloat16).float()                       # SRS: fp32 sum -> bf16
    logits = h @ w.gate_w.float().T
    p = torch.softmax(logits, dim=1)
    ex = torch.as_tensor(w.chosen, device="cuda")[sample]
    wt = torch.gather(p, 1, ex)
    wt = wt / wt.sum(1, keepdim=True)
    ref = torch.zeros_like(h)
    for s in range(k):
        for e in ex[:, s].unique().tolist():
            rows = (ex[:, s] == e).nonzero().flatten()
            x = h[rows]
            a = torch.nn.functional.silu(x @ w.w1[e].float().T) * (x @ w.w3[e].float().T)
            ref[rows] += wt[rows, s:s + 1] * (a @ w.w2[e].float().T)
    got = out[sample].float()
    err = float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))
    assert err <= TOL, err
    # per row and per element, not only in aggregate: every sampled row within
    # 2e-2 relative (row norm), every element within 2e-2 of its row's peak
    # magnitude (bf16 output + bf16 SwiGLU activations: ~4e-3 expected)
    row_err = torch.linalg.norm(got - ref, dim=1) / torch.linalg.norm(ref, dim=1)
    assert float(row_err.max()) <= 2e-2, float(row_err.max())
    peak = ref.abs().amax(dim=1, keepdim=True)
    assert float(((got - ref).abs() / peak).max()) <= 2e-2
