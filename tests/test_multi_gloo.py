"""Multi-GPU sharding logic on CPU: world_size-2 gloo process group (the GPU
compute is replaced by a deterministic stand-in runner; the sharding,
gathering, seed derivation and failure isolation are what is tested)."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2006_10509_b200.multi import Job, derived_seed, run_batch, run_sharded, shard


def fake_runner(job, device):
    if job.job_id == "bad":
        raise ValueError("broken job")
    # deterministic stand-in for a generation: depends only on the job
    return None, {"seed": job.cfg["seed"], "value": job.cfg["seed"] % 9973}


def make_jobs(n, base=42):
    jobs = [Job(f"job{i}", {"seed": derived_seed(base, f"job{i}")}, None) for i in range(n)]
    jobs.append(Job("bad", {"seed": 0}, None))
    return jobs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = run_sharded(make_jobs(n), runner=fake_runner, device_index=0)
        with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
            for r in res:
                f.write(f"{r.job_id},{r.device},{r.report['value'] if r.report else 'x'},{r.error}\n")
    finally:
        dist.destroy_process_group()


def test_shard_blocks_cover_exactly():
    for n in (0, 1, 7, 64):
        for world in (1, 2, 3, 8):
            blocks = [shard(n, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_derived_seed_matches_reference_formula():
    import hashlib

    d = hashlib.sha256(b"7:alpha").digest()
    assert derived_seed(7, "alpha") == (int.from_bytes(d[:8], "little") or 1)


def test_run_batch_is_device_count_invariant():
    jobs = make_jobs(9)
    one = run_batch(jobs, devices=[0], runner=fake_runner)
    four = run_batch(jobs, devices=[0, 1, 2, 3], runner=fake_runner)
    assert [r.job_id for r in one] == [j.job_id for j in jobs]
    assert [(r.job_id, r.report, r.error) for r in one] == [(r.job_id, r.report, r.error) for r in four]
    assert one[-1].error.startswith("ValueError")


@pytest.mark.timeout(120)
def test_gloo_world2_sharded_gather(tmp_path):
    port = _free_port()
    n = 9
    mp.spawn(_worker, args=(2, port, n, str(tmp_path)), nprocs=2, join=True)
    a = (tmp_path / "rank0.txt").read_text()
    b = (tmp_path / "rank1.txt").read_text()
    assert a == b
    lines = a.strip().splitlines()
    jobs = make_jobs(n)
    assert [ln.split(",")[0] for ln in lines] == [j.job_id for j in jobs]
    # rank 0 ran the first block, rank 1 the second (device index 0 each process)
    assert lines[-1].endswith("ValueError: broken job")
    assert all(ln.split(",")[2] == str(j.cfg["seed"] % 9973) for ln, j in zip(lines[:-1], jobs[:-1]))


# ---- OSPR subframe-shard exchange (multi._ospr_plane_exchange) on a real
# world-size-2 process group: each rank's base = sum of the lower ranks' |R|^2
# totals. Stand-in plans hold CPU planes; the all-gather is gloo.
class _PlanStandIn:
    def __init__(self, rank, shape):
        import numpy as np
        import torch

        self.shape = shape
        self.total = torch.from_numpy(np.full(shape[0] * shape[1], float(rank + 1) * 10.0 + np.arange(shape[0] * shape[1])))
        self.base = None

        class _Pb:
            precision = 1     # fp64
            device = -1       # stand-in: CPU tensors
        self.pb = _Pb()

    def copy_intensity(self, dst_ptr):
        import ctypes

        ctypes.memmove(dst_ptr, self.total.data_ptr(), self.total.numel() * 8)

    def set_intensity(self, plane_ptrs):
        import ctypes

        import numpy as np

        acc = np.zeros(self.total.numel())
        for p in plane_ptrs:
            acc += np.ctypeslib.as_array((ctypes.c_double * self.total.numel()).from_address(p))
        self.base = acc


def _ospr_worker(rank, world, port, out_dir):
    import numpy as np
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2006_10509_b200 import multi
        from paper_2006_10509_b200.slab import TorchExchange

        plan = _PlanStandIn(rank, (3, 4))
        orig_empty = torch.empty

        def cpu_empty(*a, **k):   # the exchange allocates on the plan's device; stand-in planes live on the CPU
            k.pop("device", None)
            return orig_empty(*a, **k)

        torch.empty = cpu_empty
        orig_device = torch.device
        torch.device = lambda *a, **k: orig_device("cpu")
        try:
            multi._ospr_plane_exchange([plan], TorchExchange(), [rank], world)
        finally:
            torch.empty = orig_empty
            torch.device = orig_device
        np.save(os.path.join(out_dir, f"base{rank}.npy"), plan.base)
    finally:
        dist.destroy_process_group()


def test_ospr_shard_exchange_world2_gloo(tmp_path):
    import numpy as np

    mp.spawn(_ospr_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    n = 12
    tot = [10.0 * (r + 1) + np.arange(n) for r in range(2)]
    assert np.array_equal(np.load(tmp_path / "base0.npy"), np.zeros(n))          # rank 0: no lower ranks
    assert np.array_equal(np.load(tmp_path / "base1.npy"), tot[0])               # rank 1: rank 0's total
