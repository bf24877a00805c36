"""B200-native speculative token shuffling MoE layer (arXiv 2503.04398).

Drop-in for the online path of the reference package `moesched`:
the scheduler API (`lookup_devices`, `rebatch_tokens`, `resume_tokens`,
`gate_permutation`, `apply_expert_shuffle`, `remap_topk`), the MDLB bundle
reader, the comm model / event counter, and the MoE-layer forward
(`SpecMoELayer`).  All compute runs in libsmoe.so (sm_100a); importing the
package does not need a GPU, calling it does.
"""

from .predictor import DeviceNGramTable, TokenDeviceTable, encode_history
from .scheduler import (PAD_TOKEN, GatePermutation, LookupBundle, SchedulerError,
                        ShuffleIndices, apply_expert_shuffle, bundle_memory,
                        bundle_memory_bytes, gate_permutation, lookup_device, lookup_devices,
                        rebatch_rows, rebatch_tokens, remap_topk, resume_tokens,
                        schedule_requests_dp)

__version__ = "0.1.0"


def __getattr__(name):
    # heavier modules load lazily (they touch torch / CUDA)
    if name == "SpecMoELayer":
        from .layer import SpecMoELayer
        return SpecMoELayer
    raise AttributeError(name)
