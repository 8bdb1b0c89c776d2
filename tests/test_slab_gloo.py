"""Row-distributed GS driver (config C6) under a real world-size-2 gloo group
on CPU: slab layout, corner turns (block transposes + all_to_all_single),
all-reduced error sums, gathered index plane and cancel consensus, with the
pass kernels replaced by the numpy stand-in of tests/slab_numpy_ops.py.
Checked against the oracle; the GPU kernels themselves are covered by
tests/test_gpu_slab.py."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cgh_oracle as O
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200 import slab as SL
from paper_2006_10509_b200.image import rect_mask
from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec
from paper_2006_10509_b200.workloads import gaussian_beam, natural_target

from slab_numpy_ops import NumpyOps


def _cfg(n, kind, iters, init="random-phase", mask=True, gain=0.25):
    rects = [(n // 8, n // 6, n // 2, n // 3)] if mask else []
    return A.AlgorithmConfig("gs", SlmSpec(n, n, PhaseOnly(8)), PropagationSpec(kind, distance=0.05),
                             MetricSpec(rect_mask(n, n, rects), rescale=mask), seed=11, iterations=iters,
                             feedback_gain=gain, init_mode=init)


CASES = [(32, "fresnel", 5, "random-phase", True), (64, "fourier", 4, "backpropagate", False)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        exch = SL.TorchExchange()
        lines = []
        for n, kind, iters, init, beam in CASES:
            cfg = _cfg(n, kind, iters, init)
            target = natural_target(n)
            illum = gaussian_beam(n, n) if beam else None
            holo, rep = SL.run_gs_slab(cfg, target, illum, exchange=exch,
                                       ops_factory=lambda rk, cfg=cfg, n=n: NumpyOps(cfg, n, world, rk))
            np.save(os.path.join(out_dir, f"holo_{n}_{rank}.npy"), holo)
            lines.append(f"{n} {rep.iterations_executed} {rep.termination} " +
                         " ".join(repr(e) for _, e in rep.error_trace) + f" eff {rep.efficiency!r}")

        class StopAfter:
            def __init__(self, k):
                self.k, self.calls = k, 0

            def is_set(self):   # only rank 1 asks to stop: consensus must stop both
                self.calls += 1
                return rank == 1 and self.calls > self.k

        cfg = _cfg(32, "fourier", 9)
        holo, rep = SL.run_gs_slab(cfg, natural_target(32), None, cancel=StopAfter(2), exchange=exch,
                                   ops_factory=lambda rk: NumpyOps(cfg, 32, world, rk))
        np.save(os.path.join(out_dir, f"holo_cancel_{rank}.npy"), holo)
        lines.append(f"cancel {rep.iterations_executed} {rep.termination}")
        with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
            f.write("\n".join(lines) + "\n")
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_slab_driver_world2_gloo_matches_oracle(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = (tmp_path / "rank0.txt").read_text().splitlines()
    r1 = (tmp_path / "rank1.txt").read_text().splitlines()
    assert r0 == r1   # every rank reports the same run
    for (n, kind, iters, init, beam), line in zip(CASES, r0):
        cfg = _cfg(n, kind, iters, init)
        target = natural_target(n)
        illum = gaussian_beam(n, n) if beam else None
        ref_holo, ref = O.gs(cfg, target, illum)
        parts = line.split()
        assert int(parts[1]) == iters and parts[2] == "completed"
        trace = [float(x) for x in parts[3:3 + iters + 1]]
        assert np.max(np.abs(np.array(trace) - [e for _, e in ref.error_trace]) / trace) < 1e-10
        assert abs(float(parts[-1]) - ref.efficiency) < 1e-10
        for rank in (0, 1):
            holo = np.load(tmp_path / f"holo_{n}_{rank}.npy")
            assert np.array_equal(holo, ref_holo)
    assert r0[-1] == "cancel 2 cancelled"
    ref_holo, _ = O.gs(_cfg(32, "fourier", 2), natural_target(32))
    assert np.array_equal(np.load(tmp_path / "holo_cancel_0.npy"), ref_holo)


def test_slab_layout_helpers_roundtrip():
    rows = np.arange(8 * 32).reshape(8, 32).astype(np.complex128)
    seg = SL.to_segments(rows)
    assert seg.shape == (4, 8, 8)
    assert np.array_equal(seg[2, 3], rows[3, 16:24])
    assert np.array_equal(SL.from_segments(seg), rows)


def test_local_inputs_partition_the_shifted_target():
    n, world = 16, 4
    cfg = _cfg(n, "fourier", 1)
    target = natural_target(n)
    illum = gaussian_beam(n, n)
    full = np.where(np.fft.ifftshift(cfg.metric.mask), np.abs(np.fft.ifftshift(target)),
                    -np.abs(np.fft.ifftshift(target)))
    cols = []
    for rank in range(world):
        loc, stats = SL.local_inputs(cfg, target, illum, world, rank)
        cols.append(loc["tgt"].T)
        assert np.array_equal(loc["beam"], np.abs(illum[rank * 4:(rank + 1) * 4]))
        assert stats["count_in"] == int(np.sum(cfg.metric.mask))
    got = np.concatenate(cols, axis=1)
    assert np.array_equal(got, full) and np.array_equal(np.signbit(got), np.signbit(full))
