"""Multi-GPU layer: independent holograms sharded across the GPUs of one node.

SURVEY.md §8(e). The hot path shards naturally at the hologram level
(batched targets, batched OSPR holograms): each GPU runs whole generations
with no data-path collective; only the per-job reports are gathered. SA/DBS
runs are sequential per proposal, so several GPUs run replicas (independent
seeds/targets) — "replicas only".

Two front ends:

* ``run_batch(jobs, devices)`` — one process driving several GPUs with one
  host thread per device (the C ABI releases the GIL), mirroring the
  reference's thread-pool batch runner (``controller.py:336-356``); results
  come back in job order and are identical for any device count because
  seeds are fixed per job (``derived_seed``, ``controller.py:95-97``).
* ``run_sharded(jobs, runner, group)`` — one process per GPU under
  ``torch.distributed`` (torchrun); rank r runs the contiguous block
  ``shard(len(jobs), world, r)`` and the reports are gathered to every rank
  with ``all_gather_object`` (gloo on CPU for tests, NCCL on GPUs).
"""

from __future__ import annotations

import hashlib
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field


def derived_seed(base_seed: int, job_id: str) -> int:
    """Per-job seed from (batch base seed, job id) — controller.py:95-97."""
    digest = hashlib.sha256(f"{base_seed}:{job_id}".encode("utf-8")).digest()
    return int.from_bytes(digest[:8], "little") or 1


def shard(n_items: int, world: int, rank: int):
    """Contiguous block [start, stop) of ``n_items`` owned by ``rank``."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return start, stop


@dataclass
class Job:
    """One generation: config, target, optional illumination, job id."""

    job_id: str
    cfg: object
    target: object
    illumination: object = None
    meta: dict = field(default_factory=dict)


@dataclass
class JobResult:
    job_id: str
    report: object = None
    hologram: object = None
    error: str | None = None
    device: int | None = None


def _default_runner(job, device_index):
    from .algorithms import RUNNERS
    from .runtime import device

    with device(device_index):
        return RUNNERS[job.cfg.algorithm](job.cfg, job.target, job.illumination)


def run_batch(jobs, devices=(0,), runner=None, keep_holograms=True):
    """Run ``jobs`` on ``devices`` (one host thread per device); a failing job
    is recorded and does not abort the batch (controller.py:328-333)."""
    runner = runner or _default_runner
    devices = list(devices)
    if not devices:
        raise ValueError("need at least one device")
    buckets = [[] for _ in devices]
    for i, _ in enumerate(jobs):
        buckets[i % len(devices)].append(i)
    results = [None] * len(jobs)

    def work(slot):
        dev = devices[slot]
        for i in buckets[slot]:
            job = jobs[i]
            try:
                holo, rep = runner(job, dev)
                results[i] = JobResult(job.job_id, rep, holo if keep_holograms else None, None, dev)
            except Exception as exc:  # noqa: BLE001 - per-job isolation like the reference
                results[i] = JobResult(job.job_id, None, None, f"{type(exc).__name__}: {exc}", dev)

    with ThreadPoolExecutor(max_workers=len(devices)) as pool:
        list(pool.map(work, range(len(devices))))
    return results


def run_sharded(jobs, runner=None, group=None, device_index=None, keep_holograms=False):
    """torch.distributed sharding: this rank runs its contiguous block of jobs;
    returns all ranks' results (job order) on every rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    runner = runner or _default_runner
    dev = rank if device_index is None else device_index
    start, stop = shard(len(jobs), world, rank)
    mine = []
    for job in jobs[start:stop]:
        try:
            holo, rep = runner(job, dev)
            mine.append(JobResult(job.job_id, rep, holo if keep_holograms else None, None, dev))
        except Exception as exc:  # noqa: BLE001
            mine.append(JobResult(job.job_id, None, None, f"{type(exc).__name__}: {exc}", dev))
    if world == 1:
        return mine
    gathered = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    return [r for part in gathered for r in part]
