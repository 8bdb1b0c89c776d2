"""Multi-GPU layer: independent holograms sharded across the GPUs of one node.

SURVEY.md §8(e). The hot path shards naturally at the hologram level
(batched targets, batched OSPR holograms): each GPU runs whole generations
with no data-path collective; only the per-job reports are gathered. SA/DBS
runs are sequential per proposal, so several GPUs run replicas (independent
seeds/targets) — "replicas only".

Three front ends:

* ``run_batch(jobs, devices)`` — one process driving several GPUs with one
  host thread per device (the C ABI releases the GIL), mirroring the
  reference's thread-pool batch runner (``controller.py:336-356``); results
  come back in job order and are identical for any device count because
  seeds are fixed per job (``derived_seed``, ``controller.py:95-97``).
* ``run_sharded(jobs, runner, group)`` — one process per GPU under
  ``torch.distributed`` (torchrun); rank r runs the contiguous block
  ``shard(len(jobs), world, r)`` and the reports are gathered to every rank
  with ``all_gather_object`` (gloo on CPU for tests, NCCL on GPUs).
* ``run_ospr_sharded(cfg, target, exchange=...)`` — ONE ``run_ospr`` with its
  S subframes split into contiguous parts over the ranks:
  each rank generates its part (index planes), publishes its |R|^2 total, and
  re-accumulates from the sum of the lower ranks' totals (one exchange step:
  read through peer pointers with symmetric memory, or NCCL all-gather) so the
  cumulative per-frame errors equal the single-GPU run's.
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


def device_runners(devices=(0,)):
    """Runner table for the reference's own batch driver (controller.run_batch,
    controller.py:336-356, which calls RUNNERS through controller.execute,
    controller.py:207-210): every worker thread of its ThreadPoolExecutor is
    bound to one of ``devices`` on its first call (round robin) and keeps it.

    ``cghkit.algorithms.RUNNERS.update(device_runners(range(n_gpus)))`` turns
    ``run_batch(jobs, workers=k * n_gpus, ...)`` into a multi-GPU batch while
    the manifest parsing, per-job derived seeds (controller.py:95-97), error
    rows (controller.py:328-333) and the manifest-ordered CSV
    (controller.py:348-355) stay the reference's. Holograms do not depend on the
    device count: each job's seed is fixed by (base seed, job id)."""
    import itertools
    import threading

    from .algorithms import DBS, GS, OSPR, RUNNERS, SA
    from .runtime import device

    devices = list(devices)
    if not devices:
        raise ValueError("need at least one device")
    counter = itertools.count()
    lock = threading.Lock()
    local = threading.local()

    def dev_of_thread():
        d = getattr(local, "dev", None)
        if d is None:
            with lock:
                d = devices[next(counter) % len(devices)]
            local.dev = d
        return d

    def wrap(alg):
        base = RUNNERS[alg]

        def runner(cfg, target, illumination=None, **kw):
            with device(dev_of_thread()):
                return base(cfg, target, illumination, **kw)

        runner.__name__ = base.__name__
        runner.__doc__ = base.__doc__
        return runner

    return {alg: wrap(alg) for alg in (GS, SA, DBS, OSPR)}


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


def _ospr_plane_exchange(plans, exch, rank_ids, world, cache=None):
    """Phase-1 totals -> each rank's base = sum of the lower ranks' totals.

    SimulatedExchange: the planes are the other virtual ranks' intensity
    buffers (same device). SymmetricExchange: each rank copies its total into
    a symmetric plane; after a device barrier the base kernel reads the lower
    ranks' planes through NVLink peer pointers. Otherwise (NCCL/gloo): all-gather
    into a (G, H, W) tensor and sum its first rank planes on the device."""
    import torch

    from .slab import NcclExchange, SimulatedExchange, SymmetricExchange, TorchExchange

    if isinstance(exch, NcclExchange):   # the library's NCCL all-gather on the pass stream
        (p,) = plans
        rank = rank_ids[0]
        n_el = p.shape[0] * p.shape[1]
        dt = torch.float64 if p.pb.precision == 1 else torch.float32
        dev = torch.device("cuda", p.pb.device)
        mine = torch.empty(n_el, dtype=dt, device=dev)
        p.copy_intensity(mine.data_ptr())
        allp = torch.empty((world, n_el), dtype=dt, device=dev)
        exch.all_gather_into(allp, mine)
        torch.cuda.synchronize(dev)
        p.set_intensity([allp[i].data_ptr() for i in range(rank)])
        return
    if not isinstance(exch, TorchExchange):   # LocalExchange / SimulatedExchange: all ranks in this process
        # the base of rank r reads ranks 0..r-1 before any rank overwrites its
        # own plane, so stage copies first
        n_el = plans[0].shape[0] * plans[0].shape[1]
        dt = torch.float64 if plans[0].pb.precision == 1 else torch.float32
        dev = torch.device("cuda", plans[0].pb.device)
        stage = []
        for p in plans:
            t = torch.empty(n_el, dtype=dt, device=dev)
            p.copy_intensity(t.data_ptr())
            stage.append(t)
        for r, p in zip(rank_ids, plans):
            p.set_intensity([stage[i].data_ptr() for i in range(r)])
        return
    (p,) = plans
    rank = rank_ids[0]
    n_el = p.shape[0] * p.shape[1]
    dt = torch.float64 if p.pb.precision == 1 else torch.float32
    dev = torch.device("cuda", p.pb.device)
    if isinstance(exch, SymmetricExchange):
        import torch.distributed._symmetric_memory as symm

        cache = {} if cache is None else cache
        if "symm" not in cache:   # one symmetric plane per session (rendezvous is a collective)
            plane = symm.empty(n_el, dtype=dt, device=dev)
            group = exch.group if exch.group is not None else exch.dist.group.WORLD
            cache["symm"] = (plane, symm.rendezvous(plane, group))
        plane, h = cache["symm"]
        p.copy_intensity(plane.data_ptr())
        h.barrier(channel=0)
        p.set_intensity(list(h.buffer_ptrs)[:rank])
        h.barrier(channel=0)                 # peers finished reading this rank's plane
        return
    mine = torch.empty(n_el, dtype=dt, device=dev)
    p.copy_intensity(mine.data_ptr())
    allp = torch.empty(world * n_el, dtype=dt, device=dev)   # flat: what every backend's all-gather accepts
    exch.dist.all_gather_into_tensor(allp, mine, group=exch.group)
    p.set_intensity([allp[i * n_el:(i + 1) * n_el].data_ptr() for i in range(rank)])


class OsprShardSession:
    """Prepared subframe-sharded OSPR run (plans and target resident);
    ``run()`` = phase 1, the exchange of |R|^2 totals, phase 2."""

    def __init__(self, cfg, target, illumination=None, *, exchange=None, precision=None, device=None):
        import numpy as np

        from .algorithms import _check_inputs
        from .plan import GenerationPlan
        from .slab import LocalExchange, SimulatedExchange

        target = np.asarray(target, dtype=np.complex128)
        _check_inputs(cfg, target, illumination)
        self.cfg, self.shape = cfg, target.shape
        self.exch = exchange or LocalExchange()
        self.world = self.exch.world
        self.S = int(cfg.subframes)
        self.rank_ids = list(range(self.world)) if isinstance(self.exch, SimulatedExchange) else \
            [getattr(self.exch, "rank", 0)]
        self.parts = [shard(self.S, self.world, r) for r in self.rank_ids]
        self.plans = []
        self._xcache = {}
        for _ in self.rank_ids:
            p = GenerationPlan(cfg, target.shape, precision=precision, device=device)
            p.set_target(target, illumination, amplitude_only=True)   # OSPR: no backpropagation start
            self.plans.append(p)

    def run(self, seed=None):
        """Returns (this process's per-frame errors [(k, err)], efficiency or None)."""
        import numpy as np

        streams = np.random.SeedSequence(self.cfg.seed if seed is None else seed).spawn(self.S)   # algorithms.py:487
        for p, (lo, hi) in zip(self.plans, self.parts):
            if hi > lo:
                p.ospr_part(streams[lo:hi], lo, self.S, 1)
            else:
                p.set_intensity([])
        _ospr_plane_exchange(self.plans, self.exch, self.rank_ids, self.world, self._xcache)
        trace, eff = [], None
        for p, (lo, hi) in zip(self.plans, self.parts):
            if hi > lo:
                rep, tr = p.ospr_part(streams[lo:hi], lo, self.S, 2)
                trace += tr
                if hi == self.S:
                    eff = float(rep.efficiency)
        return trace, eff

    def indices(self):
        import numpy as np

        return [p.download_indices(hi - lo) if hi > lo else np.empty((0,) + self.shape, np.uint8)
                for p, (lo, hi) in zip(self.plans, self.parts)]

    def close(self):
        for p in self.plans:
            p.close()


def run_ospr_sharded(cfg, target, illumination=None, *, exchange=None, gather=True, precision=None, device=None):
    """``run_ospr`` (algorithms.py:473-530) with the subframes sharded over
    ranks. Returns (list of complex128 subframe holograms — all S when
    ``gather``, else this rank's part —, RunReport) on every rank."""
    import time

    from .algorithms import COMPLETED, RunReport
    from .slab import SimulatedExchange
    from .slm import states

    start = time.perf_counter()
    sess = OsprShardSession(cfg, target, illumination, exchange=exchange, precision=precision, device=device)
    try:
        local_trace, eff = sess.run()
        idx_parts = sess.indices()
    finally:
        sess.close()
    exch, world = sess.exch, sess.world
    if isinstance(exch, SimulatedExchange) or world == 1:
        traces, effs, idxs = [local_trace], [eff], idx_parts
    else:
        import torch.distributed as dist

        got = [None] * world
        dist.all_gather_object(got, (local_trace, eff, idx_parts[0] if gather else None), group=exch.group)
        traces = [g[0] for g in got]
        effs = [g[1] for g in got]
        idxs = [g[2] for g in got] if gather else idx_parts
    trace = sorted((k, e) for tr in traces for k, e in tr)
    eff = next(e for e in effs if e is not None)
    table = states(cfg.slm.scheme)
    holos = [table[i] for part in idxs for i in part]
    return holos, RunReport(error_trace=trace, final_error=trace[-1][1], efficiency=eff, iterations_executed=sess.S,
                            runtime_ms=(time.perf_counter() - start) * 1e3, seed_used=cfg.seed, termination=COMPLETED)
