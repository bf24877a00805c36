"""ctypes binding of libsmoe.so (the C-ABI declared in include/smoe.h).

The product path has no CPU fallback: every compute entry point goes through
this library, and `lib()` raises if the library is missing or the current
device cannot run sm_100a code.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libsmoe.so"
_lib = None

c_i32, c_i64, c_sz, c_vp = C.c_int32, C.c_int64, C.c_size_t, C.c_void_p
P = C.c_void_p  # every device pointer crosses the boundary as a plain address

# (name, restype, argtypes) — mirrors include/smoe.h one to one.
SIGNATURES = [
    ("smoe_version", C.c_char_p, []),
    ("smoe_status_string", C.c_char_p, [C.c_int]),
    ("smoe_device_ok", C.c_int, []),
    ("smoe_set_option", C.c_int, [c_i32, c_i32]),
    ("smoe_get_option", C.c_int, [c_i32]),
    ("smoe_lookup_devices", C.c_int,
     [P, c_i64, P, c_i32, P, P, c_i64, P, P, c_i64, c_i32, P, P, P]),
    ("smoe_plan_workspace_bytes", c_sz, [c_i64, c_i32]),
    ("smoe_rebatch_plan", C.c_int, [P, c_i64, c_i32, P, P, P, P, P, P, c_sz, P]),
    ("smoe_lookup_plan", C.c_int,
     [P, c_i64, P, c_i32, P, P, c_i64, P, P, c_i64, c_i32, P, P, P, P, P, P, P, c_sz, P]),
    ("smoe_gather_rows", C.c_int, [P, c_i64, c_i32, c_i64, P, c_i64, c_i32, c_i64, P, P, P]),
    ("smoe_gate_permutation", C.c_int, [P, c_i32, c_i32, P, P, P, P]),
    ("smoe_permute_columns", C.c_int, [P, c_i64, c_i32, c_i32, P, P, P]),
    ("smoe_remap_index", C.c_int, [P, c_i64, P, c_i64, P, P, P]),
    ("smoe_count_local", C.c_int, [P, c_i64, c_i32, P, c_i32, P, P, P, P]),
    ("smoe_event_metrics", C.c_int, [P, P, c_i64, c_i32, P, c_i32, P, c_i32, P, P, P, P]),
    ("smoe_ceo_sample_scores", C.c_int, [P, c_i32, c_i32, P, P, c_i32, c_i32, P, P, P]),
    ("smoe_schedule_requests_dp", C.c_int, [P, c_i64, c_i32, P, P]),
    ("smoe_layer_workspace_bytes", c_sz, [P]),
    ("smoe_layer_create", C.c_int, [P, P]),
    ("smoe_layer_destroy", None, [P]),
    ("smoe_layer_bind", C.c_int, [P, c_i32, c_i32, P]),
    ("smoe_layer_set_tables", C.c_int, [P, P, P, c_i64, P, P, c_i64, c_i32, P]),
    ("smoe_layer_set_weights", C.c_int, [P, P, P, P, P]),
    ("smoe_layer_set_pipeline", C.c_int, [P, c_i32, c_i64]),
    ("smoe_layer_set_weights_tiled", C.c_int, [P, P, P, P, P]),
    ("smoe_tile_weights", C.c_int, [P, c_i64, c_i64, P, P]),
    ("smoe_srs", C.c_int, [P, c_i32, c_i32, c_i32, P, P, P, c_i64, c_i32, P, P]),
    ("smoe_sag", C.c_int, [P, c_i32, P, P, P, c_i64, c_i32, P, c_i32, P]),
    ("smoe_pack_w13", C.c_int, [P, P, c_i32, c_i32, c_i32, P, P]),
    ("smoe_layer_stage", C.c_int, [P, c_i32, P, P, c_i64, P]),
    ("smoe_layer_forward", C.c_int, [P, P, P, c_i64, P]),
    ("smoe_layer_stage_hist", C.c_int, [P, c_i32, P, P, c_i32, c_i32, c_i64, P]),
    ("smoe_layer_forward_hist", C.c_int, [P, P, P, c_i32, c_i32, c_i64, P]),
    ("smoe_layer_barrier", C.c_int, [P, P]),
    ("smoe_gate_topk", C.c_int,
     [P, c_i64, c_i32, P, P, c_i32, c_i32, c_i32, P, c_i32, P, P, P, P]),
    ("smoe_pair_offsets", C.c_int, [P, c_i64, c_i32, c_i32, P, P, P]),
    ("smoe_pack_rows", C.c_int, [P, c_i64, c_i32, c_i32, P, P, P]),
    ("smoe_combine_rows", C.c_int, [P, P, P, c_i64, c_i32, c_i32, P, P]),
    ("smoe_grouped_gemm", C.c_int,
     [P, c_i64, c_i64, P, c_i64, c_i64, P, c_i32, c_i32, P, c_i64, c_i64, P]),
    ("smoe_device_alloc", C.c_int, [c_sz, P]),
    ("smoe_device_free", C.c_int, [P]),
    ("smoe_ipc_handle", C.c_int, [P, P]),
    ("smoe_ipc_open", C.c_int, [P, P]),
    ("smoe_ipc_close", C.c_int, [P]),
]

# status codes / error bits / enums (include/smoe.h)
OK, ERR_INVALID_ARG, ERR_LENGTH, ERR_UNSUPPORTED, ERR_CUDA, ERR_CLUSTERS, ERR_GATE_WIDTH = range(7)
ERRBIT_DEVICE_RANGE = 1
ERRBIT_EXPERT_LABEL = 2
ERRBIT_TOKEN_RANGE = 4
ERRBIT_HISTORY_RANGE = 8
ERRBIT_INDEX_RANGE = 16
ERRBIT_CAPACITY = 32
ERRBIT_TIMEOUT = 64
MAX_SHARDS = 16
OPT_GEMM_CTA_GROUP_UP, OPT_GEMM_CTA_GROUP_DOWN, OPT_GATE_TENSOR = 0, 1, 2
OPT_GEMM_PAIR_MIN_ROWS = 3
OPT_PDL = 4
OPT_PDL_STAGES = 5
OPT_GEMM_NARROW_MAX_ROWS = 6
OPT_DEDUP_DISPATCH = 7
OPT_EARLY_DOWN = 8
OPT_ROUTE_IN_GATE = 9
OPT_GEMM_GROUP_M_UP = 10
OPT_GEMM_GROUP_M_DOWN = 11
OPT_DECODE_UP_PDL = 12

(BUF_PARTIAL, BUF_XIN, BUF_XMETA, BUF_YPAIR, BUF_OUT, BUF_COUNTS, BUF_SIGNAL, BUF_HS,
 BUF_TOPK_IDS, BUF_TOPK_W, BUF_PAIR_RANK, BUF_HMID, BUF_FORWARD, BUF_INVERSE, BUF_DEV,
 BUF_PLAN_COUNTS, BUF_GROUP, BUF_STATS, BUF_ERR, BUF_WORKSPACE, BUF_PROBLEMS,
 BUF_EPOCH, BUF_HIST_OUT, BUF_XFAN, BUF_AR, BUF_AG) = range(26)
PIPELINE_SMOE, PIPELINE_DSMOE = 0, 1
(STAT_LOCAL_PAIRS, STAT_REMOTE_PAIRS, STAT_SRS_ROWS, STAT_GROUP, STAT_REMOTE_ROWS,
 STAT_SENT_ROWS) = range(6)
STAT_COUNT = 16
(STAGE_PLAN, STAGE_SRS, STAGE_GATE, STAGE_ROUTE, STAGE_DISPATCH, STAGE_EXPERT_UP,
 STAGE_EXPERT_DOWN, STAGE_COMBINE_SAG) = range(8)
STAGE_NAMES = ("plan", "srs", "gate", "route", "dispatch", "expert_up", "expert_down",
               "combine_sag")


class LayerConfig(C.Structure):
    _fields_ = [("n_shards", c_i32), ("shard_begin", c_i32), ("shard_count", c_i32),
                ("n_experts", c_i32), ("top_k", c_i32), ("hidden", c_i32), ("ffn", c_i32),
                ("renormalize", c_i32), ("max_tokens", c_i64), ("expert_rows", c_i64),
                ("world_size", c_i32), ("world_rank", c_i32)]


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


def load(path: str | os.PathLike | None = None):
    """dlopen libsmoe.so and declare every signature (no device needed)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # SMOE_LIB: an alternative in-tree build (A/B experiments between builds)
    p = Path(path) if path else Path(os.environ.get("SMOE_LIB", _LIB_PATH))
    if not p.exists():
        raise ImportError(f"{p} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    handle = C.CDLL(str(p))
    for name, res, args in SIGNATURES:
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = handle
    return handle


_device_checked = False


def lib():
    """The library, after checking that the current CUDA device is sm_100."""
    global _device_checked
    h = load()
    if not _device_checked:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2503_04398_b200 needs a CUDA device (B200, sm_100a); "
                               "there is no CPU fallback")
        torch.cuda.init()
        if not h.smoe_device_ok():
            raise RuntimeError("current CUDA device is not sm_100 (B200); kernels are sm_100a only")
        _device_checked = True
    return h


def check(status: int, what: str = "") -> None:
    if status != OK:
        msg = load().smoe_status_string(status).decode()
        raise NativeError(f"{what or 'smoe call'} failed: {msg} (status {status})")


def ptr(t) -> int:
    """Device address of a torch tensor (0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
