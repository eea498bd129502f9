"""bench.py's N>1 path (torchrun, one process per rank, barrier + max-over-
ranks timing, per-step scale-gradient exchange, rank-0 JSON line) on the one
GPU of the box: two ranks share cuda:0 with the gloo backend
(--dist-backend gloo, a test-only switch; the scaling run uses NCCL with one
GPU per rank)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_gloo():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--dist-backend", "gloo", "--steps", "6", "--warmup", "3", "--no-cpu", "--no-secondary",
           "--e2e-steps", "3"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]   # rank 0 prints exactly one line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 6
    assert d["e2e"]["value"] > 0
    assert "frames sharded over 2 GPU" in d["config"]["parallelism"]
