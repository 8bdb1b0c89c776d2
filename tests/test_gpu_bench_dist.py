"""bench.py under torchrun with one rank, forced onto the collective code paths
(CGHB200_BENCH_FORCE_DIST=1): NCCL process group, symmetric-memory exchanges of
the C6 slab run and of the sharded OSPR run, barriers and max-over-ranks. Guards
the N > 1 paths of the driver's scaling run on a single GPU."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_collective_paths_single_rank():
    env = dict(os.environ, CGHB200_BENCH_FORCE_DIST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", "29517", os.path.join(REPO, "bench.py"), "--gpus", "1", "--no-cpu",
           "--no-search", "--no-c5", "--no-e2e", "--no-hgi", "--steps", "3", "--no-fp64"]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=REPO)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert "error" not in line["c6"] and line["c6"]["value"] > 0, line["c6"]
    assert "cgh_multi" in line["c6"]["exchange"], line["c6"]["exchange"]   # the library data plane
    assert "cgh_multi" in line["ospr_sharded"]["exchange"], line["ospr_sharded"]["exchange"]
    assert "error" not in line["ospr_sharded"] and line["ospr_sharded"]["value"] > 0, line["ospr_sharded"]
