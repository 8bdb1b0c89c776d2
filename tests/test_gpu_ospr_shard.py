"""run_ospr with its subframes sharded over G ranks (multi.run_ospr_sharded,
SURVEY.md §8(e) C2), G virtual ranks on one device (SimulatedExchange):
subframe holograms identical to the single-GPU run_ospr (generation does not
depend on the exchanged intensity), cumulative traces and efficiency equal
up to summation order; C2 at full size against the reference's golden trace."""

import numpy as np
import pytest

import golden_cases as G
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.image import rect_mask
from paper_2006_10509_b200.multi import run_ospr_sharded
from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
from paper_2006_10509_b200.runtime import precision
from paper_2006_10509_b200.slab import SimulatedExchange
from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec, binary_phase, states
from paper_2006_10509_b200.workloads import natural_target

pytestmark = pytest.mark.gpu


def _cfg(n, kind, scheme, frames, mask):
    rects = [(n // 8, n // 8, n // 2, n // 3)] if mask else []
    return A.AlgorithmConfig("ospr", SlmSpec(n, n, scheme), PropagationSpec(kind, distance=0.05),
                             MetricSpec(rect_mask(n, n, rects), rescale=mask), seed=4, subframes=frames)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("n,kind,scheme,frames,mask,world", [
    (256, "fourier", binary_phase(), 8, False, 2),
    (512, "fresnel", PhaseOnly(4), 6, True, 3),
    (1024, "fourier", binary_phase(), 7, False, 4),
    (256, "fourier", PhaseOnly(8), 3, False, 1),
])
def test_sharded_ospr_matches_single_gpu(prec, n, kind, scheme, frames, mask, world):
    cfg = _cfg(n, kind, scheme, frames, mask)
    target = natural_target(n)
    with precision(prec):
        ref_h, ref = A.run_ospr(cfg, target)
        got_h, rep = run_ospr_sharded(cfg, target, exchange=SimulatedExchange(world) if world > 1 else None)
    assert len(got_h) == frames
    assert all(np.array_equal(a, b) for a, b in zip(got_h, ref_h))
    assert [k for k, _ in rep.error_trace] == [k for k, _ in ref.error_trace]
    e1 = np.array([e for _, e in rep.error_trace])
    e0 = np.array([e for _, e in ref.error_trace])
    tol = 1e-5 if prec == "fp32" else 1e-12
    assert np.max(np.abs(e1 - e0) / e0) < tol
    assert abs(rep.efficiency - ref.efficiency) < tol


def test_c2_sharded_over_4_against_golden():
    name = "C2_ospr_1024_bin_24"
    rec = G.manifest()["cases"][name]
    cfg, target, illum = G.build(rec)
    arrs = G.load_arrays(name)
    with precision("fp32"):
        holos, rep = run_ospr_sharded(cfg, target, illum, exchange=SimulatedExchange(4))
    tr = np.array([e for _, e in rep.error_trace])
    assert np.max(np.abs(tr - arrs["trace"]) / arrs["trace"]) < 1e-3
    assert abs(rep.efficiency - rec["efficiency"]) < 1e-4
    table = states(cfg.slm.scheme)
    for i in (0, len(holos) - 1):
        assert np.sum(holos[i] != table[arrs[f"idx{i}"]]) <= 64


def _symm_worker(proc, out_path):
    import torch
    import torch.distributed as dist

    from paper_2006_10509_b200.slab import SymmetricExchange

    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = _cfg(512, "fresnel", PhaseOnly(4), 5, True)
        with precision("fp32"):
            holos, rep = run_ospr_sharded(cfg, natural_target(512), exchange=SymmetricExchange())
        np.save(out_path, np.stack(holos))
        np.save(out_path + ".trace.npy", np.array([e for _, e in rep.error_trace] + [rep.efficiency]))
    finally:
        dist.destroy_process_group()


def test_sharded_ospr_symmetric_memory_single_rank(tmp_path):
    """Peer-plane exchange (symmetric memory rendezvous + device barriers) on
    a one-rank NCCL group equals run_ospr."""
    import os
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(s.getsockname()[1])
    s.close()
    out = str(tmp_path / "h.npy")
    mp.spawn(_symm_worker, args=(out,), nprocs=1, join=True)
    cfg = _cfg(512, "fresnel", PhaseOnly(4), 5, True)
    with precision("fp32"):
        ref_h, ref = A.run_ospr(cfg, natural_target(512))
    assert np.array_equal(np.load(out), np.stack(ref_h))
    got = np.load(out + ".trace.npy")
    want = np.array([e for _, e in ref.error_trace] + [ref.efficiency])
    assert np.max(np.abs(got - want) / want) < 1e-5
