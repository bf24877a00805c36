"""bench.py --impl reference: JSON contract, and every timed step runs the
calibrated sample (the reported tokens are the tokens the oracle processed)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def test_reference_arm_json_line():
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--config", "toy", "--steps", "2", "--warmup", "1", "--cpu-budget", "0.5"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == "MoE-layer tokens/sec" and line["higher_is_better"] is True
    assert line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"]
    ns = line["config"]["tokens_per_step"]
    # value is consistent with the per-step time of ns tokens
    assert np.isclose(line["value"], ns / (line["ms_per_step"] / 1e3), rtol=1e-6)


def test_oracle_sample_fixed_runs_that_many_tokens(monkeypatch):
    import bench
    from oracle import layer_ref
    from paper_2503_04398_b200 import synth
    seen = []
    orig = layer_ref.layer_forward

    def spy(**kw):
        seen.append(len(kw["tokens"]))
        return orig(**kw)
    monkeypatch.setattr(layer_ref, "layer_forward", spy)
    w = synth.make_workload("toy", n=300, eps=0.2, seed=3, device=False)
    ns, _ = bench.oracle_sample(w.bundle, w.partials, w.tokens, w.hist, w.gate_w, w.w1, w.w3,
                                w.w2, 2, 0.0, 300, fixed=200)
    assert ns == 200 and seen == [200]
