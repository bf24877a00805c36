"""Host <-> device plumbing shared by the API mirror (torch = allocator + streams)."""

from __future__ import annotations

import numpy as np

from . import _native


def torch():
    import torch as _t
    return _t


def is_torch(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor)


def device():
    return torch().device("cuda", torch().cuda.current_device())


_NP_TO_TORCH = None


def _np_to_torch_dtype(dt: np.dtype):
    global _NP_TO_TORCH
    t = torch()
    if _NP_TO_TORCH is None:
        _NP_TO_TORCH = {
            np.dtype(np.int8): t.int8, np.dtype(np.uint8): t.uint8,
            np.dtype(np.int16): t.int16, np.dtype(np.uint16): t.uint16,
            np.dtype(np.int32): t.int32, np.dtype(np.uint32): t.uint32,
            np.dtype(np.int64): t.int64, np.dtype(np.uint64): t.uint64,
            np.dtype(np.float16): t.float16, np.dtype(np.float32): t.float32,
            np.dtype(np.float64): t.float64, np.dtype(np.bool_): t.bool,
        }
    if dt not in _NP_TO_TORCH:
        raise TypeError(f"dtype {dt} is not supported by the device path")
    return _NP_TO_TORCH[dt]


def to_device(x, dtype=None):
    """numpy / list / torch -> contiguous CUDA tensor (copy only when needed)."""
    t = torch()
    if isinstance(x, t.Tensor):
        y = x
        if dtype is not None and y.dtype != dtype:
            y = y.to(dtype)
        if y.device.type != "cuda":
            y = y.to(device())
        return y.contiguous()
    a = np.ascontiguousarray(np.asarray(x))
    _np_to_torch_dtype(a.dtype)            # rejects dtypes the device path cannot hold
    y = t.from_numpy(a).to(device(), non_blocking=False)
    if dtype is not None and y.dtype != dtype:
        y = y.to(dtype)
    return y


def to_host_like(y, like):
    """Return torch tensors as-is for torch callers, numpy for everyone else."""
    if is_torch(like):
        return y
    return y.cpu().numpy()


# Deferred error mode (scheduler.defer_errors): every call ORs its error bits
# into one sticky device flag per device instead of its own, and nothing is
# read back until scheduler.check_errors() -- no host synchronisation per call.
_DEFER = {"on": False, "flags": {}}


def sticky_flag():
    t = torch()
    dev = device()
    f = _DEFER["flags"].get(str(dev))
    if f is None:
        f = t.zeros(1, dtype=t.int32, device=dev)
        _DEFER["flags"][str(dev)] = f
    return f


class ErrFlag:
    """Device int32 error flag read back after a call (one small D2H), or, in
    deferred mode, a view of the sticky per-device flag."""

    def __init__(self, allow_defer: bool = False):
        t = torch()
        self.deferred = allow_defer and _DEFER["on"]
        self.t = sticky_flag() if self.deferred else t.zeros(1, dtype=t.int32, device=device())

    @property
    def ptr(self) -> int:
        return _native.ptr(self.t)

    def bits(self) -> int:
        return int(self.t.item())
