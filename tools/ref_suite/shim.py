"""Run the REFERENCE's own test suite with its online-path modules swapped
for this package (the drop-in check of INTEGRATION.md §2).

    python tools/ref_suite/shim.py <copy-of-reference-pkg> [pytest args]

`<copy-of-reference-pkg>` is a copy of /root/reference/pkg (src/ + tests/),
made by the caller (tools/ref_suite/run_on_gpu.sh copies it next to the repo
snapshot; nothing under it is committed).  The reference package is imported
from that copy, then every name the online path owns is replaced by this
package's -- the GPU implementations behind libsmoe.so:

  moesched.scheduler  lookup_devices, lookup_device, rebatch_tokens,
                      resume_tokens, gate_permutation, apply_expert_shuffle,
                      remap_topk, schedule_requests_dp, bundle_memory(_bytes),
                      LookupBundle, ShuffleIndices, GatePermutation,
                      SchedulerError, PAD_TOKEN
  moesched.comm       simulate_layer, simulate_trace (event counts on the GPU)
                      and the volume model (volume_collective ... sweep_alpha)
  moesched.solver     metrics (smoe_event_metrics)
  moesched.tables     read_bundle, write_bundle, export_token_csv, TableError

(also re-bound on the top-level `moesched` package).  Profiling, predictor
builders, the solver search and the CLI stay the reference's: they are the
offline toolkit, out of scope, and several tests drive the
swapped functions through them (e.g. cli simulate -> comm.simulate_trace).
The tests themselves run unmodified.
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]

SWAP = {
    "scheduler": ("lookup_devices", "lookup_device", "rebatch_tokens", "resume_tokens",
                  "gate_permutation", "apply_expert_shuffle", "remap_topk",
                  "schedule_requests_dp", "bundle_memory", "bundle_memory_bytes", "LookupBundle",
                  "ShuffleIndices", "GatePermutation", "SchedulerError", "PAD_TOKEN"),
    "comm": ("simulate_layer", "simulate_trace", "volume_collective", "pipeline_volume",
             "dense_pipeline", "sharded_pipeline", "tensor_parallel_pipeline", "saving_ratio",
             "sweep_alpha", "vanilla_token_labels", "Stage", "PipelineSpec", "VolumeReport",
             "CommError", "MODES"),
    "solver": ("metrics", "SolverError"),
    "tables": ("read_bundle", "write_bundle", "export_token_csv", "TableError"),
}


def install(ref_src: Path) -> dict:
    """Import the reference from `ref_src` and swap in our implementations.
    Returns {module: [names swapped]}."""
    sys.path.insert(0, str(ref_src))
    sys.path.insert(0, str(ROOT))
    import importlib
    import moesched
    ours = importlib.import_module("paper_2503_04398_b200")
    done = {}
    for mod, names in SWAP.items():
        ref_mod = importlib.import_module(f"moesched.{mod}")
        our_mod = importlib.import_module(f"paper_2503_04398_b200.{mod}")
        for name in names:
            obj = getattr(our_mod, name)
            setattr(ref_mod, name, obj)
            if hasattr(moesched, name):
                setattr(moesched, name, obj)
        done[mod] = list(names)
    moesched.__b200_shim__ = ours.__name__
    return done


class _Plugin:
    def __init__(self, swapped):
        self.swapped = swapped

    def pytest_report_header(self, config):
        return [f"moesched online path swapped for paper_2503_04398_b200: "
                f"{ {k: len(v) for k, v in self.swapped.items()} } names"]


def main(argv):
    import pytest
    pkg = Path(argv[0]).resolve()
    swapped = install(pkg / "src")           # before the reference's conftest imports moesched
    args = argv[1:] or [str(pkg / "tests"), "-q", "-p", "no:cacheprovider"]
    return pytest.main(args + ["--rootdir", str(pkg)], plugins=[_Plugin(swapped)])


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
