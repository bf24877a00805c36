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
