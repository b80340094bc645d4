"""The N > 1 path of bench.py / the trainer, run functionally on one GPU: two
torchrun ranks on the same device with the gloo backend (SAL_DIST_BACKEND).  The
gradient all-reduce cannot be captured under gloo, so this also exercises the
split pre/post step graphs.  Not a measurement."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REPO = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(*args, timeout=600):
    env = dict(os.environ, SAL_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(REPO / "bench.py"),
           "--gpus", "2", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]   # rank 0 prints exactly one line
    return json.loads(lines[0])


def test_two_rank_training_bench_line():
    d = _torchrun("--shape", "arxiv", "--steps", "12", "--warmup", "3", "--no-cpu-baseline",
                  "--kernel-batches", "3")
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2"
    assert d["config"]["global_batch"] == 2048
    # arxiv: 90,941 train ids -> 89 batches -> 45 steps per rank at W = 2
    assert d["config"]["steps_per_epoch"] == 45
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0


def test_two_rank_inference_and_reference_arm():
    d = _torchrun("--mode", "infer", "--shape", "arxiv", "--warmup", "3")
    assert d["n_gpus"] == 2 and d["config"]["steps_per_rank"] == 24   # 48,603 ids / 1024 / 2
    assert d["e2e"]["total"] == 48603
    r = _torchrun("--impl", "reference", "--shape", "arxiv", "--steps", "2", "--warmup", "1",
                  "--cpu-seconds", "2")
    assert r["impl"] == "reference" and r["n_gpus"] == 2
