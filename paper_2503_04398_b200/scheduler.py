"""Online token scheduling on the GPU — drop-in for `moesched.scheduler`.

Same names, argument meaning, return types and exceptions as the reference
module (`/root/reference/pkg/src/moesched/scheduler.py`); the arithmetic runs
in the sm_100a kernels of libsmoe.so through the C-ABI (include/smoe.h).
numpy inputs give numpy outputs; CUDA tensors stay on the device.

    lookup_devices     scheduler.py:82-98    -> smoe_lookup_devices   (K1)
    rebatch_tokens     scheduler.py:119-149  -> smoe_rebatch_plan + smoe_gather_rows
    resume_tokens      scheduler.py:152-157  -> smoe_gather_rows
    gate_permutation   scheduler.py:200-210  -> smoe_gate_permutation
    apply_expert_shuffle scheduler.py:213-219 -> smoe_permute_columns
    remap_topk         scheduler.py:222-224  -> smoe_remap_index
"""

from __future__ import annotations

import weakref
import zlib
from dataclasses import dataclass

import numpy as np

from . import _dev, _native
from .predictor import DeviceNGramTable, TokenDeviceTable, encode_history

PAD_TOKEN = -1


class SchedulerError(ValueError):
    pass


@dataclass(frozen=True)
class LookupBundle:
    """𝒯/𝒯p token table, 𝒜/𝒜p n-gram table and ℰ expert labels
    (scheduler.py:24-38)."""

    token_table: TokenDeviceTable
    ngram_table: DeviceNGramTable
    expert_labels: np.ndarray
    layers: int

    def __post_init__(self):
        object.__setattr__(self, "expert_labels", np.asarray(self.expert_labels, dtype=np.int16))
        if self.token_table.n_clusters != self.ngram_table.n_clusters:
            raise SchedulerError("table cluster counts disagree")


@dataclass(frozen=True)
class ShuffleIndices:
    forward: np.ndarray      # original position of each shuffled slot, -1 pad
    inverse: np.ndarray      # shuffled slot of each original position
    group_size: int
    n_devices: int

    @property
    def n_tokens(self) -> int:
        return len(self.inverse)


@dataclass(frozen=True)
class GatePermutation:
    new_to_old: np.ndarray
    old_to_new: np.ndarray
    n_clusters: int


def bundle_memory_bytes(vocab: int, n_clusters: int, n: int, layers: int,
                        n_experts: int | None = None) -> dict:
    """Serving footprint (scheduler.py:41-52): int16 token labels per layer,
    E^n rows of E float32 probabilities + an int16 best label, int16 ℰ."""
    token = 2 * vocab * layers
    ngram = (n_clusters ** n) * (4 * n_clusters + 2)
    expert = 2 * (n_experts or 0)
    return {"token_table": token, "ngram_table": ngram, "expert_table": expert,
            "total": token + ngram + expert}


def bundle_memory(bundle) -> dict:
    return bundle_memory_bytes(vocab=len(bundle.token_table.labels),
                               n_clusters=bundle.token_table.n_clusters,
                               n=bundle.ngram_table.n, layers=bundle.layers,
                               n_experts=len(bundle.expert_labels))


# ---------------------------------------------------------------- device tables
class DeviceTables:
    """The lookup tables resident in HBM (int16 labels, float32 confidences).

    `best`/`confidence` of the n-gram table are taken from the table's own
    properties, so the device copy is bit-identical to what the reference's
    lookup compares (predictor.py:72-78)."""

    def __init__(self, bundle):
        t = _dev.torch()
        tok = bundle.token_table
        ng = bundle.ngram_table
        self.n_clusters = int(tok.n_clusters)
        self.vocab = int(len(tok.labels))
        self.t_labels = _dev.to_device(np.asarray(tok.labels, dtype=np.int16))
        self.t_conf = _dev.to_device(np.asarray(tok.confidence, dtype=np.float32))
        best = np.asarray(ng.best, dtype=np.int16)
        conf = np.asarray(ng.confidence, dtype=np.float32)
        self.a_rows = int(len(conf))
        self.a_best = _dev.to_device(best if best.size else np.zeros(1, np.int16))
        self.a_conf = _dev.to_device(conf if conf.size else np.zeros(1, np.float32))
        self.ngram_n = int(ng.n)
        del t


# id(bundle) -> (weakref to the bundle, content fingerprint, DeviceTables).
# Entries die with their bundle (weakref callback), and a bundle whose arrays
# were edited in place since the upload is re-uploaded (fingerprint).
_TABLE_CACHE: dict[int, tuple[weakref.ref, int, DeviceTables]] = {}


def _fingerprint(bundle) -> int:
    tok, ng = bundle.token_table, bundle.ngram_table
    h = 0
    for a in (tok.labels, tok.confidence, ng.best, ng.confidence):
        a = np.ascontiguousarray(np.asarray(a))
        h = zlib.adler32(memoryview(a).cast("B"), h)
    return h


def device_tables(bundle) -> DeviceTables:
    key = id(bundle)
    fp = _fingerprint(bundle)
    hit = _TABLE_CACHE.get(key)
    if hit is not None and hit[0]() is bundle and hit[1] == fp:
        return hit[2]
    dt = DeviceTables(bundle)
    try:
        ref = weakref.ref(bundle, lambda _r, k=key: _TABLE_CACHE.pop(k, None))
    except TypeError:                       # not weak-referenceable: do not cache
        return dt
    _TABLE_CACHE[key] = (ref, fp, dt)
    return dt


def defer_errors(on: bool = True):
    """Deferred error reporting for device-resident callers: while on, the
    scheduler functions do not read their error flag back after each call
    (which synchronises the host with the device); the kernels OR their bits
    into a sticky per-device flag that `check_errors()` reads, resets and
    raises from (SchedulerError / IndexError, as the immediate mode would).
    rebatch_tokens still synchronises: its output size depends on the
    device-computed group size (scheduler.py:136).  Usable as a context
    manager: `with defer_errors(): ...; check_errors()`."""
    prev = _dev._DEFER["on"]
    _dev._DEFER["on"] = bool(on)

    class _Ctx:
        def __enter__(self):
            return self

        def __exit__(self, *exc):
            _dev._DEFER["on"] = prev
            return False
    return _Ctx()


def check_errors() -> None:
    """Raise (and clear) the errors accumulated in deferred mode."""
    f = _dev.sticky_flag()
    bits = int(f.item())
    f.zero_()
    _raise_for(bits)


def _check(err) -> None:
    if not err.deferred:
        _raise_for(err.bits())


def _raise_for(bits: int, index_msg: str = "index out of range") -> None:
    if bits & _native.ERRBIT_DEVICE_RANGE:
        raise SchedulerError("device label out of range")
    if bits & _native.ERRBIT_EXPERT_LABEL:
        raise SchedulerError("expert label out of range")
    if bits & (_native.ERRBIT_TOKEN_RANGE | _native.ERRBIT_HISTORY_RANGE
               | _native.ERRBIT_INDEX_RANGE):
        raise IndexError(index_msg)


# ---------------------------------------------------------------- lookup
def lookup_devices(bundle, tokens, histories):
    """Device of each token: the n-gram prediction when its confidence
    strictly exceeds the token's threshold, else the static label."""
    L = _native.lib()
    tabs = device_tables(bundle)
    tok = _dev.to_device(tokens, _dev.torch().int64).reshape(-1)
    n = tok.numel()
    out = _dev.torch().empty(n, dtype=_dev.torch().int64, device=tok.device)
    hist = None
    hist_len = 0
    if histories is not None:
        hist = _dev.to_device(histories, _dev.torch().int64)
        if hist.dim() != 2:
            raise IndexError("histories must be (n_tokens, n)")
        if hist.shape[0] != n:
            raise IndexError("histories do not align with tokens")
        hist_len = int(hist.shape[1])
    if n == 0:
        return _dev.to_host_like(out, tokens)
    err = _dev.ErrFlag(allow_defer=True)
    _native.check(L.smoe_lookup_devices(
        _native.ptr(tok), n, _native.ptr(hist), hist_len, _native.ptr(tabs.t_labels),
        _native.ptr(tabs.t_conf), tabs.vocab, _native.ptr(tabs.a_best), _native.ptr(tabs.a_conf),
        tabs.a_rows, tabs.n_clusters, _native.ptr(out), err.ptr, _native.stream_ptr()),
        "lookup_devices")
    _check(err)
    return _dev.to_host_like(out, tokens)


def lookup_device(bundle, token: int, history) -> tuple[int, str]:
    """Scalar twin (scheduler.py:63-79): (device, "ngram" | "token")."""
    use_hist = history is not None and len(history) == bundle.ngram_table.n
    hist = np.asarray(history, dtype=np.int64).reshape(1, -1) if use_hist else None
    dev = int(np.asarray(lookup_devices(bundle, np.array([token], dtype=np.int64), hist))[0])
    source = "token"
    if use_hist:
        row = int(encode_history(np.asarray(history, dtype=np.int64),
                                 bundle.ngram_table.n_clusters))
        tabs = device_tables(bundle)
        conf = float(tabs.a_conf[row].item())
        thr = float(tabs.t_conf[int(token)].item())
        if conf > thr:
            source = "ngram"
    return dev, source


# ---------------------------------------------------------------- rebatch / resume
class _Plan:
    def __init__(self, devices_t, n_devices: int):
        t = _dev.torch()
        L = _native.lib()
        n = devices_t.numel()
        dev = devices_t.device
        cap = max(n, 1) * n_devices
        self.forward = t.empty(cap, dtype=t.int64, device=dev)
        self.inverse = t.empty(n, dtype=t.int64, device=dev)
        self.counts = t.empty(n_devices, dtype=t.int32, device=dev)
        self.group_t = t.empty(1, dtype=t.int64, device=dev)
        ws_bytes = int(L.smoe_plan_workspace_bytes(n, n_devices))
        ws = t.empty(ws_bytes, dtype=t.uint8, device=dev)
        err = _dev.ErrFlag(allow_defer=True)
        _native.check(L.smoe_rebatch_plan(
            _native.ptr(devices_t), n, n_devices, _native.ptr(self.forward),
            _native.ptr(self.inverse), _native.ptr(self.counts), _native.ptr(self.group_t),
            err.ptr, _native.ptr(ws), ws_bytes, _native.stream_ptr()), "rebatch_tokens")
        _check(err)
        self.group = int(self.group_t.item())
        self.forward = self.forward[: n_devices * self.group]


def _gather(src_t, idx_t, pad_negative: bool, pad_value: int):
    """dst[i] = src[idx[i]] over the leading axis (any trailing shape)."""
    t = _dev.torch()
    L = _native.lib()
    src_t = src_t.contiguous()
    n_out = idx_t.numel()
    row_shape = tuple(src_t.shape[1:])
    row_elems = int(np.prod(row_shape)) if row_shape else 1
    out = t.empty((n_out, *row_shape), dtype=src_t.dtype, device=src_t.device)
    if n_out == 0 or row_elems == 0:
        return out
    esz = src_t.element_size()
    err = _dev.ErrFlag(allow_defer=True)
    _native.check(L.smoe_gather_rows(
        _native.ptr(src_t), src_t.shape[0], esz, row_elems, _native.ptr(idx_t), n_out,
        1 if pad_negative else 0, int(pad_value), _native.ptr(out), err.ptr,
        _native.stream_ptr()), "gather_rows")
    _check(err)
    return out


def rebatch_tokens(tokens, devices, n_devices: int):
    """Group a batch device-contiguously (stable), padding every group to the
    largest one with PAD_TOKEN (scheduler.py:119-149)."""
    as_torch = _dev.is_torch(tokens)
    tok_np = None if as_torch else np.asarray(tokens)
    n_tok = tokens.shape[0] if as_torch else len(tok_np)
    dev_t = _dev.to_device(devices, _dev.torch().int64).reshape(-1)
    if n_tok != dev_t.numel():
        raise SchedulerError("tokens and devices must align")
    plan = _Plan(dev_t, int(n_devices))
    if as_torch:
        src = _dev.to_device(tokens)
        pad = PAD_TOKEN
    else:
        # np.full semantics of the reference (raises for dtypes that cannot hold -1)
        pad_arr = np.full(1, PAD_TOKEN, dtype=tok_np.dtype)
        if tok_np.dtype.itemsize not in (1, 2, 4, 8):
            raise TypeError(f"dtype {tok_np.dtype} is not supported by the device path")
        pad = int(pad_arr.view(_int_view(tok_np.dtype))[0])   # bit pattern of PAD in dtype
        src = _dev.to_device(tok_np)
    shuffled = _gather(src, plan.forward, True, pad)
    if as_torch:
        idx = ShuffleIndices(forward=plan.forward, inverse=plan.inverse,
                             group_size=plan.group, n_devices=int(n_devices))
        # the plan kernel's per-group counts ride along for the standalone
        # collectives (collectives._plan_tensors), so they need no recount
        object.__setattr__(idx, "_counts_t", plan.counts)
        return shuffled, idx
    idx = ShuffleIndices(forward=plan.forward.cpu().numpy(), inverse=plan.inverse.cpu().numpy(),
                         group_size=plan.group, n_devices=int(n_devices))
    return shuffled.cpu().numpy(), idx


def _int_view(dt: np.dtype):
    return {1: np.int8, 2: np.int16, 4: np.int32, 8: np.int64}[dt.itemsize]


def rebatch_rows(rows, indices: ShuffleIndices):
    """Hidden-row permutation (K2): Y[s] = X[forward[s]], zero rows for pads.
    The reference only permutes ids; this is the [n, d] matrix shuffle the
    paper fuses into SRS."""
    src = _dev.to_device(rows)
    fwd = _dev.to_device(indices.forward, _dev.torch().int64)
    out = _gather(src, fwd, True, 0)
    return _dev.to_host_like(out, rows)


def resume_tokens(shuffled, indices: ShuffleIndices):
    """Drop the padding and restore the original order (scheduler.py:152-157)."""
    n_sh = shuffled.shape[0] if _dev.is_torch(shuffled) else len(np.asarray(shuffled))
    if n_sh != len(indices.forward):
        raise SchedulerError("shuffled batch does not match the indices")
    src = _dev.to_device(shuffled)
    inv = _dev.to_device(indices.inverse, _dev.torch().int64)
    out = _gather(src, inv, False, 0)
    return _dev.to_host_like(out, shuffled)


# ---------------------------------------------------------------- s-EG
def gate_permutation(expert_labels, n_clusters: int) -> GatePermutation:
    """Cluster-contiguous expert relabelling, stable inside a cluster."""
    L = _native.lib()
    t = _dev.torch()
    lab = _dev.to_device(expert_labels, t.int64).reshape(-1)
    N = lab.numel()
    n2o = t.empty(N, dtype=t.int64, device=lab.device)
    o2n = t.empty(N, dtype=t.int64, device=lab.device)
    err = _dev.ErrFlag(allow_defer=True)
    _native.check(L.smoe_gate_permutation(_native.ptr(lab), N, int(n_clusters), _native.ptr(n2o),
                                          _native.ptr(o2n), err.ptr, _native.stream_ptr()),
                  "gate_permutation")
    _check(err)
    return GatePermutation(new_to_old=_dev.to_host_like(n2o, expert_labels),
                           old_to_new=_dev.to_host_like(o2n, expert_labels),
                           n_clusters=n_clusters)


def apply_expert_shuffle(gate_logits, perm: GatePermutation):
    """Permute gate output columns into the cluster-contiguous order."""
    L = _native.lib()
    src = _dev.to_device(gate_logits)
    width = src.shape[-1] if src.dim() else 0
    if src.dim() == 0 or width != len(perm.new_to_old):
        raise SchedulerError("gate width does not match the permutation")
    rows = src.numel() // max(width, 1)
    out = _dev.torch().empty_like(src)
    p = _dev.to_device(perm.new_to_old, _dev.torch().int64)
    _native.check(L.smoe_permute_columns(_native.ptr(src), rows, width, src.element_size(),
                                         _native.ptr(p), _native.ptr(out), _native.stream_ptr()),
                  "apply_expert_shuffle")
    return _dev.to_host_like(out, gate_logits)


def remap_topk(topk_experts, perm: GatePermutation):
    """Translate routed expert ids from the original to the shuffled layout."""
    L = _native.lib()
    t = _dev.torch()
    idx = _dev.to_device(topk_experts, t.int64)
    table = _dev.to_device(perm.old_to_new, t.int64)
    out = t.empty_like(idx)
    err = _dev.ErrFlag(allow_defer=True)
    _native.check(L.smoe_remap_index(_native.ptr(idx), idx.numel(), _native.ptr(table),
                                     table.numel(), _native.ptr(out), err.ptr,
                                     _native.stream_ptr()), "remap_topk")
    _check(err)
    return _dev.to_host_like(out, topk_experts)


def schedule_requests_dp(lengths, affinities, n_devices: int) -> np.ndarray:
    """Attention-DP request scheduling (scheduler.py:160-183): each request
    goes to its highest-affinity device still open in the current window of
    n_devices consecutive decisions.  Windows are independent, so the GPU runs
    one thread per window."""
    L = _native.lib()
    t = _dev.torch()
    K = len(lengths) if not _dev.is_torch(lengths) else int(lengths.shape[0])
    aff = _dev.to_device(affinities, t.float64)
    if tuple(aff.shape) != (K, int(n_devices)):
        raise SchedulerError("affinity matrix must be (n_requests, n_devices)")
    out = t.empty(K, dtype=t.int64, device=aff.device)
    _native.check(L.smoe_schedule_requests_dp(_native.ptr(aff), K, int(n_devices),
                                              _native.ptr(out), _native.stream_ptr()),
                  "schedule_requests_dp")
    return _dev.to_host_like(out, lengths)


__all__ = ["PAD_TOKEN", "SchedulerError", "LookupBundle", "ShuffleIndices", "GatePermutation",
           "bundle_memory_bytes", "bundle_memory", "lookup_device", "lookup_devices",
           "rebatch_tokens", "rebatch_rows", "resume_tokens", "gate_permutation",
           "apply_expert_shuffle", "remap_topk", "schedule_requests_dp", "device_tables"]
