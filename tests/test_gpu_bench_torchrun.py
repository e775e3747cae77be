"""bench.py's one-process-per-GPU path under torchrun, on one GPU: two ranks with the measurement-only solo
transport (collectives skipped) sharing device 0 — per-rank synthetic input with the degree all-gather,
per-rank group creation, barrier + max-over-ranks timing and the single JSON line from rank 0."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_torchrun_two_ranks_solo():
    env = dict(os.environ, MG_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--config", "c1", "--steps", "3", "--warmup", "3", "--solo-ranks", "--no-cpu-baseline",
           "--no-cold-e2e", "--tune", "stage_fold=2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["ms_per_step"] > 0
    assert "solo ranks" in d["config"]["parallelism"] and d["config"]["edges"] == 10566  # synth_graph(2708, 3.9, ...).nnz, from the degree all-gather
