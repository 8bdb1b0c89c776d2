#!/usr/bin/env python3
"""Benchmark of the hologram-generation hot path (BASELINE.json metric).

Headline workload (configs[2], C3): Fresnel Gerchberg-Saxton, 2048x2048,
PhaseOnly(8) quantisation, 200 iterations, full-plane mask, synthetic target
(SURVEY.md §8d). One step = one complete GS run (start field, 200 fused
iterations, final snap + replay error/efficiency) with the target already
resident in HBM. value = GS iterations/s summed over all ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs one process per GPU: under the driver's torchrun (WORLD_SIZE must
equal N), or, launched plainly, bench.py re-executes itself through
torch.distributed.run with N ranks (127.0.0.1 rendezvous); fewer than N
visible GPUs is an error. Each rank generates its own C3 hologram (seed
1 + rank): replicas, weak scaling, no data-path collective (the path does not
shard below one hologram at this size). The C5, C6 and
sharded-OSPR legs cover the workloads that do shard.

Extra objects on the JSON line: e2e (same metric through the drop-in
``run_gs`` with host numpy buffers), roofline (dominant pass, live CUDA-event
timing vs MEASURED_PEAKS.json), cpu_baseline (the oracle port on this host),
clocks (nvidia-smi sampled during the timed region), ospr (C2 holograms/s).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)


N_PX = 2048
ITERS = 200
LEVELS = 8
GS_BYTES_PER_PX = 36          # complex64: row pass 8+8, column pass 8+8+4
COL_BYTES_PER_PX = 20
ROW_BYTES_PER_PX = 16
OSPR_N = 1024
OSPR_S = 24
C5_N, C5_TARGETS, C5_ITERS = 4096, 64, 100   # batched GS (100 iterations)
C6_N, C6_ITERS = 16384, 20                   # distributed GS (§8d: "C6 timing may use 20 iterations")
# tests: take the collective code paths (symmetric memory / NCCL) even with one rank
FORCE_DIST = os.environ.get("CGHB200_BENCH_FORCE_DIST") == "1"
METRIC = "GS iterations/s (Fresnel 2048x2048, PhaseOnly(8), 200 iterations per run)"


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def free_port():
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launcher_argv(argv, n, port):
    """torch.distributed.run command that re-executes this script on n ranks."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def ensure_world(args, argv):
    """--gpus N: check an existing torchrun world, or spawn one. Returns an
    exit code when this process only launched the ranks, else None."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
            return 2
        return None
    if args.gpus <= 1 or args.impl == "reference":   # the reference arm runs on rank 0 alone
        return None
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus and not args.launch_check:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}", file=sys.stderr)
        return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")            # communicator lines: one per rank
    return subprocess.call(launcher_argv(argv, args.gpus, free_port()), env=env)


def launch_check():
    """--launch-check (tests, CPU): every rank joins a gloo group and rank 0
    prints the world it saw; no GPU work."""
    import torch
    import torch.distributed as dist

    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([float(rank)])
        dist.all_reduce(t)
        ranks = float(t.item())
        dist.destroy_process_group()
    else:
        ranks = 0.0
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "rank_sum": ranks}), flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_cfg(seed, n=N_PX, levels=LEVELS, kind="fresnel", algorithm="gs", iterations=ITERS, subframes=8):
    from paper_2006_10509_b200 import algorithms as A
    from paper_2006_10509_b200.image import rect_mask
    from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
    from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec

    return A.AlgorithmConfig(algorithm=algorithm, slm=SlmSpec(n, n, PhaseOnly(levels)),
                             propagation=PropagationSpec(kind), metric=MetricSpec(rect_mask(n, n), rescale=False),
                             seed=seed, iterations=iterations, subframes=subframes)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (getattr(self, "out", "") or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def cpu_baseline_gs(seconds_hint=20):
    """Oracle port (numpy, 1 core) on a bounded sample of the C3 workload:
    steady-state iterations/s from progress timestamps of a short run."""
    from oracle import cgh_oracle
    from paper_2006_10509_b200.workloads import natural_target

    m = 6
    cfg = make_cfg(1, iterations=m)
    target = natural_target(N_PX)
    stamps = []
    t0 = time.perf_counter()
    cgh_oracle.gs(cfg, target, progress=lambda k, e: stamps.append((k, time.perf_counter())))
    wall = time.perf_counter() - t0
    loop = [s for s in stamps if s[0] < m]
    rate = (loop[-1][0] - loop[0][0]) / (loop[-1][1] - loop[0][1])
    return {"value": rate, "unit": "iter/s", "cores": 1, "kind": "port",
            "sample": f"oracle/cgh_oracle.gs (numpy restatement of run_gs) at 2048^2 Fresnel PhaseOnly(8), "
                      f"{m} iterations, steady-state rate from progress timestamps (run wall {wall:.1f}s)"}


def run_reference(args):
    """--impl reference: the reference's CPU algorithm (oracle port) on all host
    cores: one independent C3 run per core (numpy releases the GIL), each step
    a bounded sample of 3 loop iterations per replica."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    from oracle import cgh_oracle
    from paper_2006_10509_b200.workloads import natural_target

    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        cores = os.cpu_count() or 1
    m = 4
    n_ref = int(os.environ.get("CGHB200_BENCH_REF_N", N_PX))   # tests shrink the plane
    target = natural_target(n_ref)

    def one(seed):
        stamps = []
        cgh_oracle.gs(make_cfg(seed, n=n_ref, iterations=m), target,
                      progress=lambda k, e: stamps.append((k, time.perf_counter())))
        loop = [s for s in stamps if s[0] < m]
        return loop[-1][0] - loop[0][0], loop[0][1], loop[-1][1]

    def step(pool, s):
        res = list(pool.map(one, [1 + s * cores + i for i in range(cores)]))
        iters = sum(r[0] for r in res)
        span = max(r[2] for r in res) - min(r[1] for r in res)
        return iters, span

    with ThreadPoolExecutor(max_workers=cores) as pool:
        for w in range(args.warmup):
            step(pool, args.steps + w)     # warm-up replicas use seeds after the timed ones
        tot_i, tot_t = 0, 0.0
        for s in range(args.steps):
            i, t = step(pool, s)
            tot_i += i
            tot_t += t
    value = tot_i / tot_t
    sample = (f"oracle port of run_gs on {cores} host threads, one C3 replica per thread, "
              f"{m - 1} loop iterations per replica per step (init/final excluded)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tot_t / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3: Fresnel GS 2048x2048 PhaseOnly(8), 200 it (bounded sample)",
                       "parallelism": f"{cores} CPU threads"},
            "cpu_baseline": {"value": value, "unit": "iter/s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    world, rank, local = dist_env()
    import torch

    torch.cuda.set_device(local)
    if world > 1 or FORCE_DIST:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")    # communicator lines: the driver's per-rank check

        import datetime

        # finite watchdog timeout: a rank that fails inside a collective leg
        # must not leave the others blocked for the default 10 minutes
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=datetime.timedelta(minutes=3))

    def barrier():
        if world > 1 or FORCE_DIST:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM)
        return float(t.item())

    from paper_2006_10509_b200 import _native
    from paper_2006_10509_b200 import algorithms as A
    from paper_2006_10509_b200.plan import GenerationPlan
    from paper_2006_10509_b200.runtime import device, precision
    from paper_2006_10509_b200.workloads import natural_target

    seed = 1 + rank
    cfg = make_cfg(seed)
    target = natural_target(N_PX)
    plan = GenerationPlan(cfg, (N_PX, N_PX), precision=_native.FP32, device=local)
    plan.set_target(target)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # > 126 MB L2

    clk = ClockSampler(local).__enter__()     # sampling starts before warm-up (nvidia-smi spin-up)
    for _ in range(args.warmup):
        plan.gs(seed=seed)
    step_ms = []
    launches = 0
    barrier()
    if True:
        t_wall = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            rep, _ = plan.gs(seed=seed)      # device_ms: CUDA events on the plan's stream
            step_ms.append(rep.device_ms)
            launches += rep.kernel_launches
        barrier()
        t_wall = time.perf_counter() - t_wall
    clk.__exit__(None, None, None)
    total_ms = max_over_ranks(sum(step_ms))
    value = world * args.steps * ITERS / (total_ms / 1000.0)
    launches = int(sum_over_ranks(launches))

    # per-pass timing (live CUDA events around each launch) for the roofline
    plan.profile(True)
    flush.zero_()
    torch.cuda.synchronize()
    plan.gs(seed=seed)
    passes = plan.profile(False)
    hw = N_PX * N_PX
    peak, peak_src = peaks()
    cand = []
    # the persistent warp-line loop (wl_loop: ITERS replay-plane passes at 20
    # B/px and ITERS - 1 hologram-plane passes at 16 B/px in one launch) when
    # it ran, else the per-pass kernels
    loop_bpp = (COL_BYTES_PER_PX * ITERS + ROW_BYTES_PER_PX * (ITERS - 1))
    for name, bpp in (("gs_loop", loop_bpp), ("col_gs", COL_BYTES_PER_PX), ("row_holo", ROW_BYTES_PER_PX)):
        ms, cnt = passes.get(name, (0.0, 0))
        if cnt:
            avg = ms / cnt
            cand.append((ms, name, bpp * hw / (avg / 1000.0) / 1e9, avg, bpp))
    cand.sort(reverse=True)
    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(cand[0][1]) if cand else None
        except Exception:  # noqa: BLE001
            traffic = None
    iter_ms = (sum(step_ms) / len(step_ms)) / ITERS
    roofline = None
    if cand:
        _, name, achieved, avg_ms, bpp = cand[0]
        kname = {"gs_loop": "wl_loop (persistent GS loop: 200 replay-plane + 199 hologram-plane passes per launch)",
                 "col_gs": "column pass", "row_holo": "row pass"}.get(name, name)
        roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": bpp * hw, "avg_launch_ms": avg_ms,
                    "per_iteration": {"bytes": GS_BYTES_PER_PX * hw, "ms": iter_ms,
                                      "achieved": GS_BYTES_PER_PX * hw / (iter_ms / 1000.0) / 1e9,
                                      "frac": GS_BYTES_PER_PX * hw / (iter_ms / 1000.0) / 1e9 / peak},
                    "passes_ms": {k: v[0] / max(1, v[1]) for k, v in passes.items()}}

    # the fp64 parity mode (complex128 passes; index planes bit-exact against
    # the reference at C3): same workload, 72 B/px algorithmic per iteration
    gs64 = None
    if not args.no_fp64:
        plan64 = GenerationPlan(cfg, (N_PX, N_PX), precision=_native.FP64, device=local)
        plan64.set_target(target)
        plan64.gs(seed=seed)                 # warm
        ms64, l64 = [], 0
        barrier()
        for _ in range(max(2, min(5, args.steps // 8))):
            flush.zero_()
            torch.cuda.synchronize()
            r64, _ = plan64.gs(seed=seed)
            ms64.append(r64.device_ms)
            l64 += r64.kernel_launches
        t64 = max_over_ranks(sum(ms64))
        it64 = sum(ms64) / len(ms64) / ITERS
        b64 = 2 * GS_BYTES_PER_PX * hw
        gs64 = {"metric": "GS iterations/s, fp64 parity mode (C3 workload in complex128)",
                "value": world * len(ms64) * ITERS / (t64 / 1000.0), "unit": "iter/s", "dtype": "f64",
                "steps": len(ms64), "ms_per_step": sum(ms64) / len(ms64), "gpu_launches_per_step": l64 / len(ms64),
                "roofline": {"bound": "hbm", "achieved": b64 / (it64 / 1000.0) / 1e9, "peak": peak, "unit": "GB/s",
                             "frac": b64 / (it64 / 1000.0) / 1e9 / peak, "algorithmic_bytes_per_iteration": b64,
                             "ms_per_iteration": it64}}
        plan64.close()

    # e2e: the drop-in run_gs with host numpy buffers (H2D target+mask, D2H indices)
    e2e = None
    if not args.no_e2e:
        with device(local), precision("fp32"):
            A.run_gs(cfg, target)       # warm
            barrier()
            t0 = time.perf_counter()
            ke = max(1, min(args.steps, 10))
            for _ in range(ke):
                A.run_gs(cfg, target)
            barrier()
            te = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": world * ke * ITERS / te, "unit": "iter/s",
               "h2d_bytes_per_step": hw * 16 + hw, "d2h_bytes_per_step": hw * 1 + (ITERS + 1) * 16,
               "note": "run_gs(cfg, numpy complex128 target) per step: H2D of target (pinned staging by 4 host "
                       "threads) + mask, D2H of the uint8 index plane, host states[idx] expansion"}

    # OSPR holograms/s, resident target: C2 (1024^2 binary, 24 subframes) and
    # the metric's 2048^2 size (binary, 24 subframes)
    ospr = None
    if not args.no_ospr:
        from paper_2006_10509_b200.slm import binary_phase, SlmSpec

        ospr = {}
        for on, key in ((OSPR_N, "c2_1024"), (N_PX, "2048")):
            ocfg = make_cfg(seed, n=on, kind="fourier", algorithm="ospr", subframes=OSPR_S)
            ocfg.slm = SlmSpec(on, on, binary_phase())
            oplan = GenerationPlan(ocfg, (on, on), precision=_native.FP32, device=local)
            oplan.set_target(natural_target(on))
            for _ in range(max(1, args.warmup)):
                oplan.ospr(seed=seed)
            barrier()
            oms = []
            olaunch = 0
            for _ in range(max(3, args.steps // 4)):
                flush.zero_()
                torch.cuda.synchronize()
                r, _ = oplan.ospr(seed=seed)
                oms.append(r.device_ms)
                olaunch += r.kernel_launches
            otot = max_over_ranks(sum(oms))
            ohw = on * on
            obytes = (33 * OSPR_S + 8) * ohw
            avg = sum(oms) / len(oms)
            ospr[key] = {"metric": f"OSPR holograms/s ({on}x{on} binary, {OSPR_S} subframes)",
                         "value": world * len(oms) / (otot / 1000.0), "unit": "holograms/s", "ms_per_hologram": avg,
                         "gpu_launches_per_hologram": olaunch / len(oms),
                         "roofline": {"bound": "hbm", "achieved": obytes / (avg / 1000.0) / 1e9, "peak": peak,
                                      "unit": "GB/s", "frac": obytes / (avg / 1000.0) / 1e9 / peak,
                                      "algorithmic_bytes": obytes}}
            oplan.close()

    # SA / DBS (C4: 1024^2 binary, seed 3): proposals/s and pixels/s, fp64 state
    search = None
    if not args.no_search:
        from paper_2006_10509_b200.slm import SlmSpec, binary_phase

        scfg = make_cfg(3 + rank, n=1024, kind="fourier", algorithm="sa")
        scfg.slm = SlmSpec(1024, 1024, binary_phase())
        scfg.proposals = 20000
        splan = GenerationPlan(scfg, (1024, 1024), precision=_native.FP64, device=local)
        splan.set_target(natural_target(1024))
        splan.sa(proposals=300)
        rs, _ = splan.sa()
        rd, _ = splan.dbs(max_passes=1)
        search = {"sa": {"metric": "SA proposals/s (1024x1024 binary, 20000 proposals, auto T0)",
                         "value": rs.iterations_executed / (rs.device_ms / 1000.0), "unit": "proposals/s",
                         "run_ms": rs.device_ms, "final_error": rs.final_error},
                  "dbs": {"metric": "DBS pixels/s (1024x1024 binary, one raster pass)",
                          "value": 1024 * 1024 / (rd.device_ms / 1000.0), "unit": "pixels/s", "run_ms": rd.device_ms,
                          "final_error": rd.final_error},
                  "cpu_reference": {"sa_proposals_per_s": "150-186 (BASELINE.md, survey container)",
                                    "dbs_pixels_per_s": "116 (BASELINE.md, survey container)"}}
        splan.close()

    # C5: batched GS, targets 1..64 (seed = target id) in contiguous blocks per
    # rank (multi.shard), a bounded sample of each rank's block timed
    c5 = None
    if not args.no_c5:
      try:
        from paper_2006_10509_b200.multi import shard
        from paper_2006_10509_b200.workloads import batched_target

        lo, hi = shard(C5_TARGETS, world, rank)
        mine = list(range(lo + 1, hi + 1))[: max(1, args.c5_sample)]
        c5cfg = make_cfg(1, n=C5_N, kind="fourier", iterations=C5_ITERS)
        c5plan = GenerationPlan(c5cfg, (C5_N, C5_N), precision=_native.FP32, device=local)
        c5plan.set_target(batched_target(C5_N, mine[0]))
        c5plan.gs(seed=mine[0], iterations=5)           # warm-up
        gen_ms, e2e_s = [], 0.0
        c5launch = 0
        for tid in mine:
            tgt = batched_target(C5_N, tid)              # host synthesis, not timed
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            c5plan.set_target(tgt)                       # H2D target + mask, device prep
            rep5, _ = c5plan.gs(seed=tid)
            c5plan.download_indices(1)                   # D2H index plane
            e2e_s += time.perf_counter() - t0
            gen_ms.append(rep5.device_ms)
            c5launch += rep5.kernel_launches
        barrier()
        n_done = int(sum_over_ranks(len(mine)))
        t5 = max_over_ranks(sum(gen_ms)) / 1000.0
        te5 = max_over_ranks(e2e_s)
        hw5 = C5_N * C5_N
        it_ms = sum(gen_ms) / len(gen_ms) / C5_ITERS
        c5 = {"metric": f"batched GS holograms/s ({C5_N}x{C5_N} Fourier PhaseOnly(8), {C5_ITERS} iterations, "
                        f"targets 1..{C5_TARGETS} sharded over ranks)",
              "value": n_done / t5, "unit": "holograms/s", "hologram_iterations_per_s": n_done * C5_ITERS / t5,
              "scaling": "weak", "targets_timed": n_done,
              "sample": f"first {len(mine)} target(s) of each rank's block of {hi - lo}",
              "gpu_launches_per_hologram": c5launch / len(mine),
              "e2e": {"value": n_done / te5, "unit": "holograms/s", "h2d_bytes_per_step": hw5 * 17,
                      "d2h_bytes_per_step": hw5, "note": "set_target (complex128 target + mask) + GS + index download"},
              "roofline": {"bound": "hbm", "achieved": GS_BYTES_PER_PX * hw5 / (it_ms / 1000.0) / 1e9, "peak": peak,
                           "unit": "GB/s",
                           "frac": GS_BYTES_PER_PX * hw5 / (it_ms / 1000.0) / 1e9 / peak,
                           "algorithmic_bytes_per_iteration": GS_BYTES_PER_PX * hw5, "ms_per_iteration": it_ms}}
        c5plan.close()
      except Exception as exc:  # noqa: BLE001 - reported in the JSON line, not fatal for the headline
        c5 = {"error": f"{type(exc).__name__}: {exc}"}

    # C6: one 16384^2 GS plane over all ranks (row slabs, block-transpose corner
    # turns, NCCL all_to_all_single between passes when N > 1)
    c6 = None
    if not args.no_c6:
      try:
        from paper_2006_10509_b200 import slab as SL

        c6cfg = make_cfg(1, n=C6_N, kind="fourier", iterations=C6_ITERS)
        target6 = natural_target(C6_N)
        exch_kind = "none (G = 1: local block transposes)"
        sess = None
        if world > 1 or FORCE_DIST:
            try:   # the library's data plane: IPC peer stores from the fused turn kernel + device barrier, NCCL sums
                sess = SL.SlabSession(c6cfg, target6, exchange=SL.NcclExchange(device=local), precision=_native.FP32,
                                      device=local)
                exch_kind = ("fused turn kernel: transposed blocks stored to CUDA-IPC-mapped peer buffers over NVLink "
                             "+ device barrier on peer flags (cgh_multi_*)")
            except Exception as exc:  # noqa: BLE001
                try:   # torch symmetric memory for the peer mappings
                    sess = SL.SlabSession(c6cfg, target6, exchange=SL.SymmetricExchange(), precision=_native.FP32,
                                          device=local)
                    exch_kind = f"fused turn kernel over torch symmetric memory (cgh_multi unavailable: {exc})"
                except Exception as exc2:  # noqa: BLE001
                    exch_kind = f"nccl all_to_all_single (peer mappings unavailable: {type(exc2).__name__}: {exc2})"
            if world > 1:   # every rank takes the same exchange
                ok = torch.tensor([1 if sess is not None else 0], dtype=torch.int32, device=f"cuda:{local}")
                dist.all_reduce(ok, op=dist.ReduceOp.MIN)
                if int(ok.item()) == 0 and sess is not None:
                    sess.close()
                    sess = None
                    exch_kind = "nccl all_to_all_single (symmetric memory unavailable on another rank)"
        if sess is None:
            sess = SL.SlabSession(c6cfg, target6, exchange=SL.TorchExchange() if world > 1 else None,
                                  precision=_native.FP32, device=local)
        del target6
        sess.run()                                       # warm-up
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c6ms = []
        for _ in range(max(1, args.c6_steps)):
            barrier()
            ev0.record()
            sums6, done6, _ = sess.run()
            ev1.record()
            torch.cuda.synchronize()
            c6ms.append(ev0.elapsed_time(ev1))
        t6 = max_over_ranks(sum(c6ms)) / 1000.0
        err6 = sess.errors(sums6, done6)
        sess.close()
        if hasattr(sess.exch, "close"):
            sess.exch.close()
        hw6 = C6_N * C6_N
        ms6 = max_over_ranks(sum(c6ms)) / len(c6ms) / C6_ITERS
        c6 = {"metric": f"distributed GS iterations/s ({C6_N}x{C6_N} Fourier PhaseOnly(8), one plane over "
                        f"{world} GPU(s), {C6_ITERS} iterations per run)",
              "value": len(c6ms) * C6_ITERS / t6, "unit": "iter/s", "scaling": "strong", "ms_per_iteration": ms6,
              "exchange": exch_kind,
              "final_error": err6[-1],
              "roofline": {"bound": "hbm", "achieved": GS_BYTES_PER_PX * hw6 / (ms6 / 1000.0) / 1e9 / world,
                           "peak": peak, "unit": "GB/s (per GPU)",
                           "frac": GS_BYTES_PER_PX * hw6 / (ms6 / 1000.0) / 1e9 / world / peak,
                           "algorithmic_bytes_per_iteration": GS_BYTES_PER_PX * hw6,
                           "note": "36 B/px algorithmic; the design also moves 2 x 16 B/px of corner turns"}}
      except Exception as exc:  # noqa: BLE001
        c6 = {"error": f"{type(exc).__name__}: {exc}"}

    # C2 OSPR with its 24 subframes sharded over the ranks (strong scaling,
    # one exchange of |R|^2 totals per hologram)
    ospr_sh = None
    if not args.no_ospr:
      try:
        from paper_2006_10509_b200.multi import OsprShardSession
        from paper_2006_10509_b200.slab import SymmetricExchange, TorchExchange
        from paper_2006_10509_b200.slm import SlmSpec as _Slm, binary_phase as _bin

        scfg2 = make_cfg(1, n=OSPR_N, kind="fourier", algorithm="ospr", subframes=OSPR_S)
        scfg2.slm = _Slm(OSPR_N, OSPR_N, _bin())
        t2 = natural_target(OSPR_N)
        kind2 = "none (1 GPU)"
        exch2 = None
        if world > 1 or FORCE_DIST:
            from paper_2006_10509_b200.slab import NcclExchange

            try:
                exch2, kind2 = NcclExchange(device=local), "library NCCL all-gather of |R|^2 totals (cgh_multi_*)"
            except Exception:  # noqa: BLE001
                try:
                    exch2, kind2 = SymmetricExchange(), "|R|^2 totals read through NVLink peer pointers"
                except Exception:  # noqa: BLE001
                    exch2, kind2 = TorchExchange(), "NCCL all-gather of |R|^2 totals"
        with device(local), precision("fp32"):
            sess2 = OsprShardSession(scfg2, t2, exchange=exch2)
            sess2.run()                                                            # warm
            reps2 = max(3, min(10, args.steps // 4))
            barrier()
            t0 = time.perf_counter()
            for _ in range(reps2):
                sess2.run()
            barrier()
            ts2 = max_over_ranks(time.perf_counter() - t0) / reps2
            sess2.close()
            if exch2 is not None and hasattr(exch2, "close"):
                exch2.close()
        ospr_sh = {"metric": f"OSPR holograms/s, one C2 hologram ({OSPR_N}x{OSPR_N} binary, {OSPR_S} subframes) "
                             f"sharded over {world} GPU(s)", "value": 1.0 / ts2, "unit": "holograms/s",
                   "scaling": "strong", "exchange": kind2,
                   "note": "wall time per hologram with plans and target resident (phase 1, exchange of |R|^2 "
                           "totals, phase 2; per-frame errors on the host), max over ranks"}
      except Exception as exc:  # noqa: BLE001
        ospr_sh = {"error": f"{type(exc).__name__}: {exc}"}

    # .hgi output: payload + CRC-32 of the C3 hologram from
    # its index plane on the device vs host expansion + zlib (serialio.py:167-185)
    hgi = None
    if not args.no_hgi:
        import zlib

        from paper_2006_10509_b200 import serialio
        from paper_2006_10509_b200.slm import states as state_table

        idx3 = plan.download_indices(1)[0]
        table3 = state_table(cfg.slm.scheme)
        serialio.hologram_payload(idx3, table3, device=local)          # warm
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            _, crc_dev = serialio.hologram_payload(idx3, table3, device=local)
        t_dev = (time.perf_counter() - t0) / reps
        t0 = time.perf_counter()
        for _ in range(reps):
            serialio.hologram_payload(idx3, table3, device=local, expand="device")
        t_devx = (time.perf_counter() - t0) / reps
        t0 = time.perf_counter()
        for _ in range(reps):
            payload = table3[idx3]
            crc_host = zlib.crc32(payload) & 0xFFFFFFFF
        t_host = (time.perf_counter() - t0) / reps
        nbytes = idx3.size * 16
        hgi = {"metric": "hgi payload + CRC-32 of the C3 hologram (2048x2048 complex128, 64 MiB)",
               "device_ms": t_dev * 1e3, "device_expand_ms": t_devx * 1e3, "host_ms": t_host * 1e3,
               "device_gb_per_s": nbytes / t_dev / 1e9,
               "host_gb_per_s": nbytes / t_host / 1e9, "crc_equal": crc_dev == crc_host,
               "note": "device: CRC-32 on the GPU from the uint8 index plane while host threads expand "
                       "states[idx] (device_expand_ms: expansion on the GPU + pageable D2H instead); "
                       "host: numpy states[idx] + zlib.crc32 (1 thread)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_gs()

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": "C3: Fresnel GS 2048x2048, PhaseOnly(8), 200 iterations per run, "
                                       "full-plane mask, natural_target, seed 1+rank",
                           "global_batch": world, "parallelism": f"replicas x{world}",
                           "l2": "256 MB device write between timed steps (excluded from step time)"},
                "gpu_launches": launches, "wall_s_timed": t_wall,
                "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk.summary(), "ospr": ospr,
                "search": search, "c5": c5, "c6": c6, "hgi": hgi, "gs_fp64": gs64,
                "ospr_sharded": ospr_sh}
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1 or FORCE_DIST:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ospr", action="store_true")
    ap.add_argument("--no-search", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-c6", action="store_true")
    ap.add_argument("--no-hgi", action="store_true")
    ap.add_argument("--no-fp64", action="store_true")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--c5-sample", type=int, default=8, help="targets timed per rank (of its block of 64/N)")
    ap.add_argument("--c6-steps", type=int, default=3)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rc = ensure_world(args, sys.argv[1:])
    if rc is not None:
        sys.exit(rc)
    if args.launch_check:
        launch_check()
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
