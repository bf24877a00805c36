"""bench.py under torchrun with 2 and 4 ranks (the driver's N > 1 launch),
exercised on one GPU: SMOE_BENCH_SAME_GPU=1 puts every rank on cuda:0 and
uses gloo for the host plumbing (NCCL refuses two ranks on one device).  The
shards then span processes exactly as on N GPUs: IPC peer buffers, signal-pad
barriers, the pipelined e2e leg, max-over-ranks timing, one JSON line."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(nproc, *bench_args):
    env = dict(os.environ, SMOE_BENCH_SAME_GPU="1", PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1", "--master-port",
           str(_port()), str(ROOT / "bench.py"), "--gpus", str(nproc), *bench_args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-4000:]     # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("nproc", [2, 4])
def test_bench_torchrun_line(nproc):
    line = _torchrun(nproc, "--config", "mixtral", "--tokens", "1024", "--steps", "4",
                     "--warmup", "3", "--no-cpu", "--no-decode")
    assert line["n_gpus"] == nproc and line["scaling"] == "weak"
    assert line["config"]["global_tokens"] == 1024 * nproc
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    # + 5 signal-pad barriers and the deduplicated dispatch's fan-out per step
    assert line["gpu_launches"] == line["steps"] * (10 + 5 + 1)
    assert 0 < line["local_activation_rate"] < 1


def test_bench_reference_arm_torchrun():
    line = _torchrun(2, "--impl", "reference", "--config", "toy", "--steps", "2", "--warmup",
                     "1", "--cpu-budget", "0.5")
    assert line["impl"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
