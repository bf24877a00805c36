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

from .comm import (CommError, PipelineSpec, Stage, VolumeReport, dense_pipeline,
                   pipeline_volume, saving_ratio, sharded_pipeline, simulate_layer,
                   simulate_trace, sweep_alpha, tensor_parallel_pipeline, vanilla_token_labels,
                   volume_collective)
from .tables import TableError, export_token_csv, read_bundle, write_bundle
from .solver import Assignment, SolverError, ceo_sample_scores, metrics

__version__ = "0.1.0"

# Names `moesched/__init__.py:6-31` exports that belong to the offline toolkit
# (profiling, predictor builders, the co-clustering search, CLI): out of scope
# for this hot path.  They fail with a pointer, not a NameError.
_OFFLINE = frozenset((
    "EmbeddingTable", "ProfileError", "RequestTrace", "TokenExpertMatrix", "Topology",
    "ingest_profile", "emit_profile", "matrices_from_trace", "read_embeddings", "split_trace",
    "synthesize_embeddings", "synthesize_planted_profile", "validate", "write_embeddings",
    "TokenExpertConfidence", "activation_kurtosis", "build_confidence_table",
    "build_ngram_table", "evaluate_predictor", "extrapolate_oov", "token_table_from_assignment",
    "ObjectiveValue", "SolverConfig", "baseline_round_robin", "baseline_two_stage_kmeans",
    "check_constraints", "objective", "sample_labels", "solve_alternating", "solve_bruteforce",
    "solve_ceo"))


def __getattr__(name):
    # heavier modules load lazily (they touch torch / CUDA)
    if name == "SpecMoELayer":
        from .layer import SpecMoELayer
        return SpecMoELayer
    if name == "MicroBatchedSpecMoE":
        from .layer import MicroBatchedSpecMoE
        return MicroBatchedSpecMoE
    if name == "DSMoELayer":
        from .baseline import DSMoELayer
        return DSMoELayer
    if name == "DSMoEPipelineLayer":
        from .baseline import DSMoEPipelineLayer
        return DSMoEPipelineLayer
    if name in _OFFLINE:
        raise AttributeError(f"moesched.{name} is part of the offline toolkit (profiling / "
                             "solver search / CLI), out of scope for the B200 online path "
                             "(DESIGN.md §8): keep importing it from moesched")
    raise AttributeError(name)
