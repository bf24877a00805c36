"""tcgen05 grouped GEMM (K6) against a torch fp32 reference of the same op."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2503_04398_b200 import _native as N


@pytest.fixture(params=[1, 2], ids=["cta_group1", "cta_group2"], autouse=True)
def cta_group(request):
    """Run every GEMM test with the one-SM and the SM-pair MMA variants."""
    lib = N.lib()
    old = [lib.smoe_get_option(k) for k in (N.OPT_GEMM_CTA_GROUP_UP, N.OPT_GEMM_CTA_GROUP_DOWN)]
    for k in (N.OPT_GEMM_CTA_GROUP_UP, N.OPT_GEMM_CTA_GROUP_DOWN):
        N.check(lib.smoe_set_option(k, request.param), "set_option")
    yield request.param
    for k, v in zip((N.OPT_GEMM_CTA_GROUP_UP, N.OPT_GEMM_CTA_GROUP_DOWN), old):
        lib.smoe_set_option(k, v)


def run_gemm(A, B, problems, n_b, epilogue, c_cols):
    lib = N.lib()
    C = torch.zeros((A.shape[0], c_cols), dtype=torch.bfloat16, device="cuda")
    pt = torch.as_tensor(np.asarray(problems, dtype=np.int64), device="cuda")
    N.check(lib.smoe_grouped_gemm(N.ptr(A), A.shape[0], A.shape[1], N.ptr(B), B.shape[0], n_b,
                                  N.ptr(pt), len(problems), epilogue, N.ptr(C), C.shape[0],
                                  c_cols, N.stream_ptr()), "grouped_gemm")
    torch.cuda.synchronize()
    return C


def rel(a, b):
    return (a.float() - b.float()).norm().item() / max(b.float().norm().item(), 1e-30)


@pytest.mark.parametrize("M,K,NB", [(128, 64, 256), (128, 256, 256), (300, 512, 512),
                                    (1000, 1024, 768)])
def test_single_problem_store(M, K, NB):
    torch.manual_seed(M + K)
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(NB, K, device="cuda").to(torch.bfloat16)
    C = run_gemm(A, B, [[0, M, 0, 0]], NB, 0, NB)
    ref = A.float() @ B.float().T
    assert rel(C, ref) < 1e-2


def test_grouped_ragged_store():
    torch.manual_seed(1)
    K, NB, E = 512, 256, 5
    ms = [0, 1, 129, 256, 77]
    offs = np.concatenate([[0], np.cumsum(ms)])[:-1]
    A = torch.randn(int(sum(ms)) + 16, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(E * NB, K, device="cuda").to(torch.bfloat16)
    probs = [[int(offs[e]), ms[e], e, int(offs[e])] for e in range(E)]
    C = run_gemm(A, B, probs, NB, 0, NB)
    for e in range(E):
        if ms[e] == 0:
            continue
        a = A[offs[e]:offs[e] + ms[e]].float()
        ref = a @ B[e * NB:(e + 1) * NB].float().T
        assert rel(C[offs[e]:offs[e] + ms[e]], ref) < 1e-2, e
    # rows not owned by any problem stay untouched
    assert torch.count_nonzero(C[int(sum(ms)):]) == 0


def test_swiglu_epilogue():
    torch.manual_seed(2)
    E, f, d = 3, 256, 512
    ms = [200, 64, 333]
    offs = np.concatenate([[0], np.cumsum(ms)])[:-1]
    X = (torch.randn(int(sum(ms)), d, device="cuda") / 4).to(torch.bfloat16)
    w1 = (torch.randn(E, f, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
    w3 = (torch.randn(E, f, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
    w13 = torch.empty(E, 2 * f, d, dtype=torch.bfloat16, device="cuda")
    lib = N.lib()
    N.check(lib.smoe_pack_w13(N.ptr(w1), N.ptr(w3), E, f, d, N.ptr(w13), N.stream_ptr()), "pack")
    probs = [[int(offs[e]), ms[e], e, int(offs[e])] for e in range(E)]
    H = run_gemm(X, w13.view(E * 2 * f, d), probs, 2 * f, 1, f)
    for e in range(E):
        x = X[offs[e]:offs[e] + ms[e]].float()
        g = x @ w1[e].float().T
        u = x @ w3[e].float().T
        ref = torch.nn.functional.silu(g) * u
        assert rel(H[offs[e]:offs[e] + ms[e]], ref) < 1e-2, e


def test_tile_weights_layout():
    """smoe_tile_weights: box (rb, kb) = rows [256 rb, +256) x cols [64 kb, +64),
    one contiguous run, boxes ordered rb-major."""
    lib = N.lib()
    rows, cols = 512, 192
    src = torch.randn(rows, cols, device="cuda").to(torch.bfloat16)
    dst = torch.empty_like(src)
    N.check(lib.smoe_tile_weights(N.ptr(src), rows, cols, N.ptr(dst), N.stream_ptr()), "tile")
    want = src.view(rows // 256, 256, cols // 64, 64).permute(0, 2, 1, 3).reshape(rows, cols)
    assert torch.equal(dst.view(-1), want.contiguous().view(-1))
    assert lib.smoe_tile_weights(N.ptr(src), 100, cols, N.ptr(dst), N.stream_ptr()) != N.OK


def test_layer_tiled_weights_bit_identical_to_row_major(monkeypatch):
    """Box-tiled expert weights change only where the GEMMs' TMA reads from."""
    from paper_2503_04398_b200 import SpecMoELayer, synth
    over = {"G": 4, "N": 16, "k": 2, "d": 512, "f": 384}
    w = synth.make_workload("toy", n=700, eps=0.3, seed=5, cfg_override=over)
    parts = torch.from_numpy(w.partials).to(torch.bfloat16)
    outs = []
    for untiled in ("0", "1"):
        monkeypatch.setenv("SMOE_UNTILED_WEIGHTS", untiled)
        layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=700)
        assert layer.w_tiled == (untiled == "0")
        outs.append(layer.forward(parts, w.tokens, w.hist).clone())
    assert torch.equal(outs[0], outs[1])


def test_small_batch_down_gemm_single_sm_matches_pair():
    """Decode-sized batches run the down GEMM on one SM per tile; the output is
    bit-identical to the SM-pair kernel (SMOE_OPT_GEMM_PAIR_MIN_ROWS = 0)."""
    from paper_2503_04398_b200 import SpecMoELayer, synth
    lib = N.lib()
    over = {"G": 4, "N": 16, "k": 2, "d": 512, "f": 384}
    w = synth.make_workload("toy", n=64, eps=0.3, seed=6, cfg_override=over)
    parts = torch.from_numpy(w.partials).to(torch.bfloat16)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=64)
    old = lib.smoe_get_option(N.OPT_GEMM_PAIR_MIN_ROWS)
    outs = []
    try:
        for rows in (64, 0):
            N.check(lib.smoe_set_option(N.OPT_GEMM_PAIR_MIN_ROWS, rows), "opt")
            outs.append(layer.forward(parts, w.tokens, w.hist).clone())
    finally:
        N.check(lib.smoe_set_option(N.OPT_GEMM_PAIR_MIN_ROWS, old), "opt")
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("n,narrow_rows", [(64, 16), (700, 10000)])
def test_narrow_gemm_bit_identical_to_wide(n, narrow_rows):
    """The narrow GEMM variant (32-row m-blocks, 5-stage weight ring) gives the
    same bits as the 128-row tiles: at a decode-sized batch, and forced on a
    700-token batch where experts span many 32-row m-blocks
    (SMOE_OPT_GEMM_NARROW_MAX_ROWS)."""
    from paper_2503_04398_b200 import SpecMoELayer, synth
    lib = N.lib()
    over = {"G": 4, "N": 16, "k": 2, "d": 512, "f": 384}
    w = synth.make_workload("toy", n=n, eps=0.3, seed=8, cfg_override=over)
    parts = torch.from_numpy(w.partials).to(torch.bfloat16)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=2, max_tokens=n)
    old = lib.smoe_get_option(N.OPT_GEMM_NARROW_MAX_ROWS)
    outs = []
    try:
        for rows in (narrow_rows, 0):
            N.check(lib.smoe_set_option(N.OPT_GEMM_NARROW_MAX_ROWS, rows), "opt")
            assert lib.smoe_get_option(N.OPT_GEMM_NARROW_MAX_ROWS) == rows
            outs.append(layer.forward(parts, w.tokens, w.hist).clone())
    finally:
        N.check(lib.smoe_set_option(N.OPT_GEMM_NARROW_MAX_ROWS, old), "opt")
    assert torch.equal(outs[0], outs[1])
    assert outs[0].abs().sum().item() > 0


def test_grouped_512_problems_and_limit():
    """The problem table holds up to 512 problems (DS-MoE batches every
    emulated rank's (source, expert) segments into one launch); 513 is
    rejected before any device work."""
    torch.manual_seed(7)
    K, NB, E = 128, 256, 16
    rng = np.random.default_rng(0)
    ms = rng.integers(0, 9, size=512)
    offs = np.concatenate([[0], np.cumsum(ms)])[:-1]
    A = torch.randn(int(ms.sum()) + 8, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(E * NB, K, device="cuda").to(torch.bfloat16)
    probs = [[int(offs[p]), int(ms[p]), p % E, int(offs[p])] for p in range(512)]
    C = run_gemm(A, B, probs, NB, 0, NB)
    ref = torch.zeros_like(C, dtype=torch.float32)
    for p in range(512):
        if ms[p]:
            e = p % E
            ref[offs[p]:offs[p] + ms[p]] = A[offs[p]:offs[p] + ms[p]].float() @ \
                B[e * NB:(e + 1) * NB].float().T
    assert rel(C[: int(ms.sum())], ref[: int(ms.sum())]) < 1e-2
    lib = N.lib()
    pt = torch.zeros((513, 4), dtype=torch.int64, device="cuda")
    assert lib.smoe_grouped_gemm(N.ptr(A), A.shape[0], K, N.ptr(B), B.shape[0], NB, N.ptr(pt),
                                 513, 0, N.ptr(C), C.shape[0], NB, N.stream_ptr()) != N.OK
