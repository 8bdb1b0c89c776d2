"""Parity of the pipelined complex64 GS passes (fast path, N >= 256) against the
generic passes, the oracle and the full-size golden vectors (C1, C3)."""

import os

import numpy as np
import pytest

import golden_cases as G
from oracle import cgh_oracle as O
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.image import rect_mask
from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
from paper_2006_10509_b200.runtime import precision
from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec, states
from paper_2006_10509_b200.workloads import gaussian_beam, natural_target

pytestmark = pytest.mark.gpu
MAN = G.manifest()["cases"]

# fp32 index-plane mismatches against the reference (decision-boundary pixels),
# bounded at 2x the count measured on B200 (printed by the tests; round 2:
# C1 188 of 262144, C3 184 of 4194304, C2 frames 0 and 23: 0)
C1_FP32_MISMATCH_BOUND = 2 * 188
C3_FP32_MISMATCH_BOUND = 2 * 184
C2_FP32_FRAME_BOUND = 2


def _field(cfg, target, illum=None, fast=True):
    old = os.environ.pop("CGHB200_NO_FAST", None)
    if not fast:
        os.environ["CGHB200_NO_FAST"] = "1"
    try:
        with precision("fp32"):
            return A.gs_field(cfg, target, illum)
    finally:
        os.environ.pop("CGHB200_NO_FAST", None)
        if old is not None:
            os.environ["CGHB200_NO_FAST"] = old


@pytest.mark.parametrize("h,w,kind,beam,mask,gain", [
    (256, 256, "fourier", False, False, 0.0),
    (512, 1024, "fresnel", True, True, 0.5),
    (1024, 512, "fourier", False, True, 0.0),
    (2048, 2048, "fresnel", False, False, 0.0),
    (4096, 256, "fresnel", True, False, 0.2),
])
def test_fast_matches_generic(h, w, kind, beam, mask, gain):
    rects = [(w // 8, h // 8, w // 2, h // 3)] if mask else []
    cfg = A.AlgorithmConfig("gs", SlmSpec(w, h, PhaseOnly(8)), PropagationSpec(kind),
                            MetricSpec(rect_mask(w, h, rects), rescale=mask), seed=5, iterations=6,
                            feedback_gain=gain)
    target = natural_target(w, h) if h != w else natural_target(w)
    illum = gaussian_beam(h, w) if beam else None
    i1, f1, r1, t1 = _field(cfg, target, illum, fast=True)
    i2, f2, r2, t2 = _field(cfg, target, illum, fast=False)
    assert np.linalg.norm(f1 - f2) / np.linalg.norm(f2) < 2e-5
    e1 = np.array([e for _, e in t1])
    e2 = np.array([e for _, e in t2])
    assert np.max(np.abs(e1 - e2) / e2) < 1e-5
    assert np.mean(i1 != i2) < 1e-3


def test_c1_full_size_fp32_fast_and_fp64():
    name = "C1_gs_fourier_512_pl256_100"
    rec = MAN[name]
    cfg, target, illum = G.build(rec)
    arrs = G.load_arrays(name)
    with precision("fp32"):
        holo, rep = A.run_gs(cfg, target)
    tr = np.array([e for _, e in rep.error_trace])
    assert abs(rep.final_error - rec["final_error"]) / rec["final_error"] < 1e-3
    assert np.max(np.abs(tr - arrs["trace"]) / arrs["trace"]) < 1e-3
    idx = np.argmin(np.abs(holo[..., None] - states(cfg.slm.scheme)[None, None, :]), axis=-1)
    mism = int(np.sum(idx != arrs["idx0"]))
    print(f"C1 fp32 index mismatches: {mism} / {idx.size}")
    assert mism <= C1_FP32_MISMATCH_BOUND, mism
    with precision("fp64"):
        holo64, rep64 = A.run_gs(cfg, target)
    assert np.array_equal(holo64, states(cfg.slm.scheme)[arrs["idx0"]])
    assert np.max(np.abs(np.array([e for _, e in rep64.error_trace]) - arrs["trace"]) / arrs["trace"]) < 1e-9


@pytest.mark.slow
def test_c3_full_size_fp32_and_fp64():
    """C3 (the headline config): Fresnel 2048^2, PhaseOnly(8), 200 iterations."""
    name = "C3_gs_fresnel_2048_pl8_200"
    rec = MAN[name]
    cfg, target, illum = G.build(rec)
    arrs = G.load_arrays(name)
    table = states(cfg.slm.scheme)
    with precision("fp32"):
        holo, rep = A.run_gs(cfg, target)
    tr = np.array([e for _, e in rep.error_trace])
    assert abs(rep.final_error - rec["final_error"]) / rec["final_error"] < 1e-3
    assert np.max(np.abs(tr - arrs["trace"]) / arrs["trace"]) < 1e-3
    idx32 = np.searchsorted(np.angle(table) % (2 * np.pi), np.angle(holo) % (2 * np.pi) - 1e-9)
    mism32 = int(np.sum(holo != table[arrs["idx0"]]))
    print(f"C3 fp32 index mismatches: {mism32} / {holo.size}")
    assert mism32 <= C3_FP32_MISMATCH_BOUND, mism32   # decision-boundary pixels only
    with precision("fp64"):
        holo64, rep64 = A.run_gs(cfg, target)
    mism64 = int(np.sum(holo64 != table[arrs["idx0"]]))
    assert mism64 == 0, mism64
    assert np.max(np.abs(np.array([e for _, e in rep64.error_trace]) - arrs["trace"]) / arrs["trace"]) < 1e-9
    del idx32


@pytest.mark.slow
def test_c3_per_iteration_field_fp32():
    """Per-iteration complex hologram field within 1e-4 relative L2 of the oracle."""
    name = "C3_gs_fresnel_2048_pl8_200"
    cfg, target, illum = G.build(MAN[name])
    for k in (1, 3):
        cfg.iterations = k
        _, ref = O.gs(cfg, target, keep_fields=(k,))
        _, fld, _, _ = _field(cfg, target, fast=True)
        err = np.linalg.norm(fld - ref.fields[k]) / np.linalg.norm(ref.fields[k])
        assert err < 1e-4, (k, err)


def _ospr(cfg, target, illum=None, fast=True, progress=None):
    old = os.environ.pop("CGHB200_NO_FAST", None)
    if not fast:
        os.environ["CGHB200_NO_FAST"] = "1"
    try:
        with precision("fp32"):
            return A.run_ospr(cfg, target, illum, progress=progress)
    finally:
        os.environ.pop("CGHB200_NO_FAST", None)
        if old is not None:
            os.environ["CGHB200_NO_FAST"] = old


@pytest.mark.parametrize("h,w,kind,levels,beam,mask,frames", [
    (1024, 1024, "fourier", 2, False, False, 6),
    (512, 1024, "fresnel", 4, True, True, 3),
    (2048, 512, "fourier", 8, False, True, 2),
])
def test_fast_ospr_matches_generic(h, w, kind, levels, beam, mask, frames):
    from paper_2006_10509_b200.slm import PhaseOnly as PO

    rects = [(w // 8, h // 8, w // 2, h // 3)] if mask else []
    cfg = A.AlgorithmConfig("ospr", SlmSpec(w, h, PO(levels)), PropagationSpec(kind),
                            MetricSpec(rect_mask(w, h, rects), rescale=mask), seed=9, subframes=frames)
    target = natural_target(w, h) if h != w else natural_target(w)
    illum = gaussian_beam(h, w) if beam else None
    f1, r1 = _ospr(cfg, target, illum, fast=True)
    f2, r2 = _ospr(cfg, target, illum, fast=False)
    assert len(f1) == len(f2) == frames
    mism = sum(int(np.sum(a != b)) for a, b in zip(f1, f2))
    assert mism <= max(4, h * w * frames // 20000), mism
    e1 = np.array([e for _, e in r1.error_trace])
    e2 = np.array([e for _, e in r2.error_trace])
    assert np.max(np.abs(e1 - e2) / e2) < 1e-4
    assert abs(r1.efficiency - r2.efficiency) < 1e-5
    # progress path: one subframe per launch group, carried intensity
    seen = []
    f3, r3 = _ospr(cfg, target, illum, fast=True, progress=lambda k, e: seen.append(k))
    assert seen == list(range(1, frames + 1))
    assert all(np.array_equal(a, b) for a, b in zip(f1, f3))
    assert np.max(np.abs(np.array([e for _, e in r3.error_trace]) - e1) / e1) < 1e-6


def test_c2_full_size_fp32_fast():
    name = "C2_ospr_1024_bin_24"
    rec = MAN[name]
    cfg, target, illum = G.build(rec)
    arrs = G.load_arrays(name)
    table = states(cfg.slm.scheme)
    frames, rep = _ospr(cfg, target, illum, fast=True)
    tr = np.array([e for _, e in rep.error_trace])
    assert np.max(np.abs(tr - arrs["trace"]) / arrs["trace"]) < 1e-3
    assert abs(rep.efficiency - rec["efficiency"]) < 1e-4
    for i in (0, len(frames) - 1):
        mism = int(np.sum(frames[i] != table[arrs[f"idx{i}"]]))
        print(f"C2 fp32 frame {i}: {mism} index mismatches")
        assert mism <= C2_FP32_FRAME_BOUND
