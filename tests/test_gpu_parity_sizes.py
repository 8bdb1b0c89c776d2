"""Parity at the sizes the benchmarks report (VERDICT r1 "next" #1):

* C2 (OSPR 1024^2 binary x 24) in the fp64 parity mode: every subframe's index
  plane hashes to the sha256 the real reference produced
  (tests/golden/manifest.json ``idx_sha256``; algorithms.py:493-509);
* C5 size (4096^2 GS, the fast fp32 passes fast_row_holo<4096> /
  fast_col_gs<4096> with the R2 = 16 twiddle path): per-iteration hologram
  field within 1e-4 relative L2 of the oracle (oracle/cgh_oracle.py:gs, pinned
  by the golden vectors); fp64 index plane bit-exact after 3 iterations;
* C6 sizes (8192^2 / 16384^2 slab line FFTs, 32 points per thread at 16384):
  transform-only slab passes (cgh_slab_pass modes 6 = forward, 4 = inverse)
  on sampled lines against numpy.fft in fp64;
* exact-zero illumination through the fast fp32 OSPR column pass (binary
  shortcut) and the GS snapping pass against the oracle's signed-zero result.
"""

import hashlib

import numpy as np
import pytest

import golden_cases as G
from oracle import cgh_oracle as O
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200 import slab as SL
from paper_2006_10509_b200.image import rect_mask
from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
from paper_2006_10509_b200.runtime import precision
from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec, binary_phase, states
from paper_2006_10509_b200.workloads import aperture_beam, batched_target, natural_target

pytestmark = pytest.mark.gpu
MAN = G.manifest()["cases"]
# fp32 C2 mismatches vs the reference planes: 2x the measured counts (round 2
# on B200: 1 pixel in all 24 subframes, in subframe 11)
C2_FP32_MISMATCH_TOTAL = 2
C2_FP32_MISMATCH_FRAME = 2


def _indices(frame, table):
    """Exact index plane of a hologram whose values are bitwise state members."""
    idx = np.full(frame.shape, -1, np.int64)
    for k, s in enumerate(table):
        idx[frame == s] = k
    assert np.all(idx >= 0), "hologram value outside the state table"
    return idx.astype(np.uint8 if len(table) <= 256 else np.int32)


def _sha(idx):
    return hashlib.sha256(np.ascontiguousarray(idx).tobytes()).hexdigest()


def test_c2_fp64_all_subframes_match_reference_sha256():
    name = "C2_ospr_1024_bin_24"
    rec = MAN[name]
    cfg, target, illum = G.build(rec)
    arrs = G.load_arrays(name)
    table = states(cfg.slm.scheme)
    with precision("fp64"):
        frames, rep = A.run_ospr(cfg, target, illum)
    assert len(frames) == 24
    got = [_sha(_indices(f, table)) for f in frames]
    bad = [i for i, (a, b) in enumerate(zip(got, rec["idx_sha256"])) if a != b]
    assert not bad, f"subframes differing from the reference: {bad}"
    tr = np.array([e for _, e in rep.error_trace])
    assert np.max(np.abs(tr - arrs["trace"]) / arrs["trace"]) < 1e-9
    assert abs(rep.efficiency - rec["efficiency"]) < 1e-12
    # fp32 fast path, all 24 subframes against the (reference-identical) fp64 planes
    with precision("fp32"):
        frames32, rep32 = A.run_ospr(cfg, target, illum)
    per = [int(np.sum(a != b)) for a, b in zip(frames32, frames)]
    print(f"C2 fp32 index mismatches per subframe: {per} (total {sum(per)})")
    assert sum(per) <= C2_FP32_MISMATCH_TOTAL and max(per) <= C2_FP32_MISMATCH_FRAME, per


def _c5_cfg(iters):
    n = 4096
    return A.AlgorithmConfig("gs", SlmSpec(n, n, PhaseOnly(8)), PropagationSpec("fourier"),
                             MetricSpec(rect_mask(n, n)), seed=1, iterations=iters)


@pytest.mark.slow
def test_c5_4096_fast_fp32_fields_and_fp64_indices_vs_oracle():
    target = batched_target(4096, 1)
    cfg = _c5_cfg(3)
    ref_holo, ref = O.gs(cfg, target, keep_fields=(1, 2))
    for k in (1, 2):
        with precision("fp32"):
            idx, fld, rep, trace = A.gs_field(_c5_cfg(k), target)
        err = np.linalg.norm(fld - ref.fields[k]) / np.linalg.norm(ref.fields[k])
        print(f"C5 4096^2 fp32 fast field k={k}: rel L2 {err:.3e}")
        assert err < 1e-4, (k, err)
    with precision("fp64"):
        holo64, rep64 = A.run_gs(cfg, target)
    mism = int(np.sum(holo64 != ref_holo))
    print(f"C5 4096^2 fp64 3 it: {mism} index mismatches")
    assert mism == 0
    t64 = np.array([e for _, e in rep64.error_trace])
    tref = np.array([e for _, e in ref.error_trace])
    assert np.max(np.abs(t64 - tref) / tref) < 1e-9


def _slab_ops(n, prec):
    import torch

    cfg = A.AlgorithmConfig("gs", SlmSpec(n, n, PhaseOnly(8)), PropagationSpec("fourier"),
                            MetricSpec(rect_mask(n, n)), seed=1, iterations=1)
    stream = torch.cuda.current_stream(0).cuda_stream
    return SL.NativeOps(cfg, n, 1, 0, prec, 0, stream)


@pytest.mark.parametrize("n,prec", [(8192, "fp32"), (16384, "fp32"), (8192, "fp64")])
def test_slab_line_ffts_vs_numpy(n, prec):
    """Transform-only slab passes (G = 1: plain row-major lines) on 64 sampled
    lines vs numpy.fft in fp64: forward unscaled (mode 6) and inverse scaled
    by 1/N (mode 4, the backpropagation start)."""
    import torch

    p = _native.FP64 if prec == "fp64" else _native.FP32
    ops = _slab_ops(n, p)
    try:
        gen = np.random.default_rng(n)
        lines = np.sort(gen.choice(n, size=64, replace=False))
        x = gen.normal(size=(64, n)) + 1j * gen.normal(size=(64, n))
        xin = x.astype(np.complex128 if p == _native.FP64 else np.complex64)
        tol = 1e-12 if p == _native.FP64 else 1e-5
        for mode, ref in ((SL.SLAB_FWD, np.fft.fft(xin.astype(np.complex128), axis=1)),
                          (SL.SLAB_INV, np.fft.ifft(xin.astype(np.complex128), axis=1))):
            buf = ops.empty((1, n, n))
            buf.zero_()
            buf[0, torch.from_numpy(lines).to(buf.device)] = torch.from_numpy(xin).to(buf.device)
            ops.run(mode, buf)
            got = buf[0, torch.from_numpy(lines).to(buf.device)].cpu().numpy().astype(np.complex128)
            err = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
            print(f"slab {n} {prec} mode {mode}: max line rel L2 {err.max():.3e}")
            assert err.max() < tol, (mode, err.max())
            # untouched (zero) lines stay zero
            other = int((lines[0] + 1) % n) if (lines[0] + 1) % n not in set(lines.tolist()) else None
            if other is not None:
                assert float(buf[0, other].abs().max()) == 0.0
            del buf
    finally:
        ops.close()
        torch.cuda.empty_cache()


@pytest.mark.parametrize("kind,levels", [("fourier", 2), ("fresnel", 4)])
def test_zero_beam_fast_ospr_matches_oracle(kind, levels):
    """OSPR 512^2 fp32 (fast K1/K2/K3) with an aperture beam: at the exact-zero
    beam pixels the snapped index follows the reference's signed-zero phase
    (index L/2 for second-quadrant phases); compared with the oracle there."""
    n = 512
    scheme = binary_phase() if levels == 2 else PhaseOnly(levels)
    cfg = A.AlgorithmConfig("ospr", SlmSpec(n, n, scheme), PropagationSpec(kind, distance=0.05),
                            MetricSpec(rect_mask(n, n)), seed=21, subframes=2)
    target = natural_target(n)
    illum = aperture_beam(n, n)
    zero = np.abs(illum) == 0
    ref_frames, _ = O.ospr(cfg, target, illum)
    with precision("fp32"):
        frames, _ = A.run_ospr(cfg, target, illum)
    table = states(scheme)
    for f, r in zip(frames, ref_frames):
        a, b = _indices(f, table), _indices(r, table)
        assert np.any(b[zero] == levels // 2)          # the signed-zero case occurs
        mism = int(np.sum(a[zero] != b[zero]))
        assert mism <= 2, mism                          # fp32 phase near an axis only


def test_zero_beam_gs_snap_matches_oracle_fp64():
    n = 256
    cfg = A.AlgorithmConfig("gs", SlmSpec(n, n, PhaseOnly(8)), PropagationSpec("fresnel", distance=0.05),
                            MetricSpec(rect_mask(n, n)), seed=22, iterations=4)
    target = natural_target(n)
    illum = aperture_beam(n, n)
    ref_holo, ref = O.gs(cfg, target, illum)
    with precision("fp64"):
        holo, rep = A.run_gs(cfg, target, illum)
    assert np.array_equal(holo, ref_holo)
    with precision("fp32"):
        holo32, _ = A.run_gs(cfg, target, illum)
    zero = np.abs(illum) == 0
    assert int(np.sum(holo32[zero] != ref_holo[zero])) <= 2
