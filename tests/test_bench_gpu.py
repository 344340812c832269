"""bench.py's N-rank code path (DistSolver slabs, max-over-ranks timing, end-to-end leg, one JSON line from
rank 0) run as 2 processes on one GPU over gloo (PF_BENCH_BACKEND=gloo, PF_BENCH_ONE_GPU=1: a code-path
check, never a measurement)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("transport", ["nccl", "ipc"])
def test_bench_two_ranks_code_path(transport):
    env = dict(os.environ, PF_BENCH_BACKEND="gloo", PF_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
           "--warmup", "1", "--iters", "4", "--transport", transport, "--config", "C5small"]
    pr = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert pr.returncode == 0, pr.stderr[-3000:]
    lines = [l for l in pr.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0 and d["cpu_baseline"] is None
    assert "C5small" in d["config"]["workload"] and d["config"]["flow_nodes"] == 16


def test_bench_gpus_flag_self_launches():
    """`python bench.py --gpus 2` without torchrun launches 2 ranks itself (one line, n_gpus 2)."""
    env = dict(os.environ, PF_BENCH_BACKEND="gloo", PF_BENCH_ONE_GPU="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1", "--iters",
           "2", "--no-e2e", "--config", "C5small"]
    pr = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert pr.returncode == 0, pr.stderr[-3000:]
    lines = [l for l in pr.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["n_gpus"] == 2
