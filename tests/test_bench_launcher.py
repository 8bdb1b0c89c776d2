"""bench.py --gpus N launcher (CPU): N ranks are spawned through
torch.distributed.run when the script is started plainly, an existing torchrun
world must match --gpus, and too few GPUs is a loud error."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
BENCH = os.path.join(REPO, "bench.py")


def _clean_env(**kw):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    env.update(kw)
    return env


def test_too_few_gpus_is_an_error():
    import torch

    n = max(2, torch.cuda.device_count() + 1)
    out = subprocess.run([sys.executable, BENCH, "--gpus", str(n), "--steps", "1"], capture_output=True, text=True,
                         env=_clean_env(), timeout=300, cwd=REPO)
    assert out.returncode != 0
    assert f"needs {n} visible GPUs" in out.stderr


def test_world_must_match_gpus():
    out = subprocess.run([sys.executable, BENCH, "--gpus", "1", "--steps", "1"], capture_output=True, text=True,
                         env=_clean_env(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"), timeout=300, cwd=REPO)
    assert out.returncode == 2
    assert "WORLD_SIZE=2" in out.stderr


def test_launcher_argv():
    import bench

    argv = bench.launcher_argv(["--gpus", "4", "--steps", "7"], 4, 29555)
    assert argv[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in argv and "--master-addr=127.0.0.1" in argv and "--master-port=29555" in argv
    assert argv[-4:] == ["--gpus", "4", "--steps", "7"]


def test_spawned_world_of_two_gloo():
    """The plain launch re-executes bench.py on 2 ranks (gloo, no GPU work)."""
    out = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--launch-check"], capture_output=True, text=True,
                         env=_clean_env(), timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(s) for s in out.stdout.splitlines() if s.startswith("{")]
    assert len(lines) == 1                  # rank 0 alone prints
    assert lines[0]["n_gpus"] == 2 and lines[0]["rank_sum"] == 1.0
