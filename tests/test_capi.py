"""The C-ABI library loads without a GPU and exports exactly what
include/smoe.h declares (no compute calls here)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "smoe.h"
LIB = ROOT / "paper_2503_04398_b200" / "libsmoe.so"


def declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(smoe_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        from paper_2503_04398_b200 import build
        build.build()
    return ctypes.CDLL(str(LIB))


def test_header_declares_the_api():
    names = declared()
    for must in ("smoe_lookup_devices", "smoe_rebatch_plan", "smoe_lookup_plan",
                 "smoe_gather_rows", "smoe_gate_permutation", "smoe_permute_columns",
                 "smoe_remap_index", "smoe_count_local", "smoe_layer_create",
                 "smoe_layer_forward", "smoe_grouped_gemm", "smoe_ipc_handle"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_2503_04398_b200 import _native
    bound = {s[0] for s in _native.SIGNATURES}
    assert set(declared()) == bound


def test_host_only_calls(lib):
    from paper_2503_04398_b200 import _native
    h = _native.load()
    assert h.smoe_version().decode().startswith("smoe")
    assert h.smoe_status_string(0) == b"ok"
    assert h.smoe_plan_workspace_bytes(5000, 8) >= 5000 * 4
    # argument validation happens before any device work
    assert h.smoe_rebatch_plan(None, 5, 2, None, None, None, None, None, None, 0, None) == \
        _native.ERR_INVALID_ARG
    fake = 256   # never dereferenced: the shape check fails first
    assert h.smoe_rebatch_plan(fake, 5, 0, fake, fake, fake, fake, None, fake, 1 << 20, None) == \
        _native.ERR_UNSUPPORTED
    assert h.smoe_layer_create(None, None) == _native.ERR_INVALID_ARG


def test_layer_config_struct_matches_header():
    from paper_2503_04398_b200 import _native
    text = HEADER.read_text()
    body = text[text.index("typedef struct {"):text.index("} smoe_layer_config;")]
    fields = re.findall(r"int(32|64)_t\s+(\w+);", body)
    assert [f[1] for f in fields] == [f[0] for f in _native.LayerConfig._fields_]
    for (bits, name), (fname, ctype) in zip(fields, _native.LayerConfig._fields_):
        assert ctypes.sizeof(ctype) * 8 == int(bits), name


def test_new_entry_points_validate_before_device_work(lib):
    """smoe_srs / smoe_sag / smoe_tile_weights / options reject bad arguments
    on the host (no CUDA call is made, so this runs without a GPU)."""
    from paper_2503_04398_b200 import _native as N
    h = N.load()
    fake = 256
    arr = (ctypes.c_void_p * 17)(*([fake] * 17))
    p = ctypes.cast(arr, ctypes.c_void_p)
    # too many shards, bad shard range, null plan
    assert h.smoe_srs(p, 17, 0, 1, fake, fake, fake, 10, 64, p, None) == N.ERR_INVALID_ARG
    assert h.smoe_srs(p, 4, 3, 2, fake, fake, fake, 10, 64, p, None) == N.ERR_INVALID_ARG
    assert h.smoe_srs(p, 4, 0, 4, None, fake, fake, 10, 64, p, None) == N.ERR_INVALID_ARG
    assert h.smoe_sag(p, 4, fake, fake, fake, 10, 64, p, 0, None) == N.ERR_INVALID_ARG
    assert h.smoe_sag(p, 4, fake, fake, fake, 10, 64, p, 17, None) == N.ERR_INVALID_ARG
    # tile geometry: rows % 256, cols % 64
    assert h.smoe_tile_weights(fake, 100, 64, fake, None) == N.ERR_UNSUPPORTED
    assert h.smoe_tile_weights(fake, 256, 100, fake, None) == N.ERR_UNSUPPORTED
    assert h.smoe_tile_weights(None, 256, 64, fake, None) == N.ERR_INVALID_ARG
    # options: known keys round-trip, unknown keys / values are rejected
    for key, vals in ((N.OPT_GEMM_CTA_GROUP_UP, (1, 2)), (N.OPT_GEMM_CTA_GROUP_DOWN, (1, 2)),
                      (N.OPT_GATE_TENSOR, (0, 1)), (N.OPT_GEMM_PAIR_MIN_ROWS, (0, 64, 1000)),
                      (N.OPT_PDL, (0, 1)), (N.OPT_PDL_STAGES, (0, 0xff, 0xdf)),
                      (N.OPT_GEMM_NARROW_MAX_ROWS, (0, 16, 1000))):
        old = h.smoe_get_option(key)
        for v in vals:
            assert h.smoe_set_option(key, v) == N.OK and h.smoe_get_option(key) == v
        bad = {N.OPT_GEMM_PAIR_MIN_ROWS: -1, N.OPT_PDL_STAGES: 256,
               N.OPT_GEMM_NARROW_MAX_ROWS: -1}.get(key, 7)
        assert h.smoe_set_option(key, bad) == \
            N.ERR_INVALID_ARG
        assert h.smoe_set_option(key, old) == N.OK
    assert h.smoe_set_option(99, 1) == N.ERR_INVALID_ARG and h.smoe_get_option(99) == -1
