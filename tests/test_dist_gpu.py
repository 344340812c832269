"""DistSolver (the multi-GPU driver bench.py runs over NCCL) with 2 and 3 processes on one GPU over gloo:
real slab solvers, the phase-0 / phase-1 overlap schedule on a communication stream, the residual max
over ranks and the per-rank checkpoint / resume -- all bitwise equal to the single-domain run.  The
exchange is host-staged under gloo, so no rank's kernel waits on another's (tools/dist_one_gpu.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 3])
def test_dist_solver_processes_bitwise(world, tmp_path):
    pr = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "dist_one_gpu.py"), str(world)],
                        env=dict(os.environ, CK_DIR=str(tmp_path)), capture_output=True, text=True, timeout=300)
    assert pr.returncode == 0, (pr.stdout[-2000:], pr.stderr[-3000:])
    assert f"dist_one_gpu {world} bitwise" in pr.stdout
