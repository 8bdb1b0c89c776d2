"""GPU parity of the centred transforms on shapes the power-of-two passes do
not take (csrc/anysize.cu, Bluestein line DFTs): fft2 / propagate /
propagate_inverse vs numpy's pocketfft (the reference's own FFT,
propagation.py:81-123) at the reference tests' thresholds
(tests/test_propagation.py:46-66: direct-DFT agreement and forward/inverse
identity < 1e-12, Parseval < 1e-12), odd sides included."""

import numpy as np
import pytest

from oracle import cgh_oracle as O
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200 import propagation as P
from paper_2006_10509_b200.errors import NonFiniteError, UnsupportedShapeError

pytestmark = pytest.mark.gpu


def field(shape, seed):
    gen = np.random.default_rng(seed)
    return gen.normal(size=shape) + 1j * gen.normal(size=shape)


@pytest.mark.parametrize("shape", [(5, 7), (31, 33), (3, 2), (2, 3), (16, 12), (100, 300), (135, 240), (1080, 1920),
                                   (4096, 3)])
def test_fft2_any_shape_matches_numpy(shape):
    h = field(shape, sum(shape))
    ref = np.fft.fftshift(np.fft.fft2(h, norm="ortho"))
    got = P.fft2(h, "forward")
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-12
    back = P.fft2(got, "inverse")
    assert np.max(np.abs(back - h)) / np.max(np.abs(h)) < 1e-12
    assert np.allclose(P.fft2(ref, "inverse"), np.fft.ifft2(np.fft.ifftshift(ref), norm="ortho"), rtol=0, atol=1e-12)
    e_in, e_out = np.sum(np.abs(h) ** 2), np.sum(np.abs(got) ** 2)
    assert abs(e_in - e_out) / e_in < 1e-12


def test_fft2_odd_delta_and_constant():
    """Known answers (tests/test_propagation.py:33-44) on odd sides: a centred
    delta has a flat spectrum; a constant field maps to the centre pixel."""
    h = np.zeros((5, 7), complex)
    h[0, 0] = 1.0
    got = P.fft2(h, "forward")
    assert np.allclose(got, np.full((5, 7), 1 / np.sqrt(35)), atol=1e-14)
    got = P.fft2(np.ones((5, 7), complex), "forward")
    expected = np.zeros((5, 7), complex)
    expected[2, 3] = np.sqrt(35)
    assert np.allclose(got, expected, atol=1e-12)


@pytest.mark.parametrize("kind,shape", [("fresnel", (45, 60)), ("fresnel", (33, 31)), ("fourier", (96, 200))])
def test_propagate_any_shape_matches_oracle(kind, shape):
    spec = P.PropagationSpec(kind, distance=0.05)
    h = field(shape, 7)
    got = P.propagate(h, spec)
    ref = O.to_replay(h, spec)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-12
    assert np.max(np.abs(P.propagate_inverse(got, spec) - h)) / np.max(np.abs(h)) < 1e-11


def test_fp32_any_shape_within_tolerance():
    h = field((270, 480), 3)
    ref = np.fft.fftshift(np.fft.fft2(h, norm="ortho"))
    got = P._transform(h, None, 0, precision=_native.FP32)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-5


def test_any_shape_errors_are_loud():
    h = field((5, 7), 1)
    h[2, 2] = np.nan
    with pytest.raises(NonFiniteError):
        P.fft2(h, "forward")
    with pytest.raises(UnsupportedShapeError):
        P.fft2(np.ones((5000, 6), complex), "forward")   # beyond the fp64 Bluestein lines


# ---------------------------------------------------------------- GS runners
from paper_2006_10509_b200 import algorithms as A  # noqa: E402
from paper_2006_10509_b200.image import rect_mask  # noqa: E402
from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec  # noqa: E402
from paper_2006_10509_b200.runtime import precision  # noqa: E402
from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec, binary_phase  # noqa: E402
from paper_2006_10509_b200.workloads import gaussian_beam  # noqa: E402


def _target(h, w):
    y, x = np.mgrid[0:h, 0:w]
    return np.clip(0.3 + 0.5 * np.exp(-(((x - 0.4 * w) / (0.2 * w)) ** 2 + ((y - 0.6 * h) / (0.25 * h)) ** 2)),
                   0, 1).astype(complex)


def _cfg(h, w, kind="fourier", levels=8, mask=False, gain=0.0, init="random-phase", iters=10, qe=False):
    rects = [(w // 5, h // 6, w // 2, h // 2)] if mask else []     # (x, y, w, h)
    scheme = binary_phase() if levels == 2 else PhaseOnly(levels)
    return A.AlgorithmConfig("gs", SlmSpec(w, h, scheme), PropagationSpec(kind, distance=0.05),
                             MetricSpec(rect_mask(w, h, rects), rescale=mask), seed=4, iterations=iters,
                             feedback_gain=gain, quantize_each_iteration=qe, init_mode=init)


@pytest.mark.parametrize("h,w,kind,levels,mask,gain,init,beam,qe", [
    (48, 80, "fourier", 8, False, 0.0, "random-phase", False, False),
    (45, 60, "fresnel", 2, True, 0.3, "random-phase", True, False),
    (33, 31, "fourier", 16, False, 0.0, "backpropagate", False, False),
    (100, 64, "fresnel", 4, True, 0.0, "random-phase", False, True),     # non-power-of-two rows only
    (64, 96, "fourier", 8, False, 0.2, "random-phase", False, False),    # non-power-of-two columns only
])
def test_gs_any_shape_fp64_matches_oracle(h, w, kind, levels, mask, gain, init, beam, qe):
    """run_gs on planes the radix-16 passes do not take (Bluestein line DFTs):
    fp64 traces within 1e-9 of the oracle (pocketfft rounding differs from
    Bluestein's at 1e-15), index planes equal but for decision-boundary pixels."""
    cfg = _cfg(h, w, kind, levels, mask, gain, init, qe=qe)
    target = _target(h, w)
    if init == "backpropagate":
        # a real target's backpropagated start has hologram samples whose phase
        # is set by 1e-16 rounding (chaotic for any two FFTs, see
        # test_gpu_gs.CHAOTIC); a random-phase target is well conditioned
        target = target * np.exp(2j * np.pi * np.random.default_rng(h).random((h, w)))
    illum = gaussian_beam(h, w) if beam else None
    ref_holo, ref = O.gs(cfg, target, illum)
    with precision("fp64"):
        holo, rep = A.run_gs(cfg, target, illum)
    t_ref = np.array([e for _, e in ref.error_trace])
    t_got = np.array([e for _, e in rep.error_trace])
    assert len(t_got) == len(t_ref) == cfg.iterations + 1
    assert np.max(np.abs(t_got - t_ref) / t_ref) < 1e-9
    assert np.mean(holo != ref_holo) < 2e-3
    assert abs(rep.efficiency - ref.efficiency) < 1e-9


def test_gs_any_shape_fp32_and_1080p():
    cfg = _cfg(108, 192, "fresnel", 8, iters=12)
    target = _target(108, 192)
    ref_holo, ref = O.gs(cfg, target)
    with precision("fp32"):
        holo, rep = A.run_gs(cfg, target)
    t_ref = np.array([e for _, e in ref.error_trace])
    t_got = np.array([e for _, e in rep.error_trace])
    assert np.max(np.abs(t_got - t_ref) / t_ref) < 1e-3
    assert np.mean(holo != ref_holo) < 1e-2
    # a full-HD SLM plane (1080 x 1920) runs end to end and improves
    big = _cfg(1080, 1920, "fourier", 8, iters=5)
    with precision("fp32"):
        holo, rep = A.run_gs(big, _target(1080, 1920))
    tr = [e for _, e in rep.error_trace]
    assert holo.shape == (1080, 1920) and tr[-2] < tr[0] and np.all(np.isin(holo[::97, ::89], A.states(big.slm.scheme)))


@pytest.mark.parametrize("h,w,kind,levels,mask,beam,frames", [
    (45, 60, "fourier", 2, False, False, 5),
    (33, 31, "fresnel", 8, True, True, 4),       # odd sides: ifftshift != fftshift
    (100, 64, "fourier", 4, True, False, 3),     # non-power-of-two rows only
    (64, 96, "fresnel", 2, False, False, 3),     # non-power-of-two columns only
])
def test_ospr_any_shape_fp64_matches_oracle(h, w, kind, levels, mask, beam, frames):
    """run_ospr (algorithms.py:473-530) on planes the radix-16 passes do not
    take: per-frame random-phase sub-targets drawn over the centred plane and
    ifftshifted (odd sides included), Bluestein line DFTs. Subframe index
    planes equal the oracle's but for decision-boundary pixels; cumulative
    per-frame errors and efficiency within 1e-9."""
    cfg = _cfg(h, w, kind, levels, mask)
    cfg.algorithm, cfg.subframes = "ospr", frames
    target = _target(h, w)
    illum = gaussian_beam(h, w) if beam else None
    ref_frames, ref = O.ospr(cfg, target, illum)
    with precision("fp64"):
        got_frames, rep = A.run_ospr(cfg, target, illum)
    assert len(got_frames) == len(ref_frames) == frames
    for a, b in zip(got_frames, ref_frames):
        assert a.shape == (h, w) and np.mean(a != b) < 2e-3
    t_ref = np.array([e for _, e in ref.error_trace])
    t_got = np.array([e for _, e in rep.error_trace])
    assert [k for k, _ in rep.error_trace] == [k for k, _ in ref.error_trace]
    assert np.max(np.abs(t_got - t_ref) / t_ref) < 1e-9
    assert abs(rep.efficiency - ref.efficiency) < 1e-9


def test_ospr_any_shape_fp32_and_1080p():
    cfg = _cfg(108, 192, "fresnel", 2)
    cfg.algorithm, cfg.subframes = "ospr", 6
    target = _target(108, 192)
    ref_frames, ref = O.ospr(cfg, target)
    with precision("fp32"):
        got_frames, rep = A.run_ospr(cfg, target)
    t_ref = np.array([e for _, e in ref.error_trace])
    t_got = np.array([e for _, e in rep.error_trace])
    assert np.max(np.abs(t_got - t_ref) / t_ref) < 1e-3
    assert all(np.mean(a != b) < 1e-2 for a, b in zip(got_frames, ref_frames))
    # full-HD SLM plane, 24 subframes (more than one 64-frame group is not
    # needed: the group loop is shape-independent)
    big = _cfg(1080, 1920, "fourier", 2)
    big.algorithm, big.subframes = "ospr", 24
    with precision("fp32"):
        frames, rep = A.run_ospr(big, _target(1080, 1920))
    tr = [e for _, e in rep.error_trace]
    assert len(frames) == 24 and frames[0].shape == (1080, 1920)
    assert tr[-1] < tr[0] and 0 < rep.efficiency <= 1


def test_ospr_any_shape_sharded_matches_single():
    from paper_2006_10509_b200.multi import run_ospr_sharded
    from paper_2006_10509_b200.slab import SimulatedExchange

    cfg = _cfg(45, 60, "fresnel", 4, True)
    cfg.algorithm, cfg.subframes = "ospr", 7
    target = _target(45, 60)
    with precision("fp64"):
        ref_h, ref = A.run_ospr(cfg, target)
        got_h, rep = run_ospr_sharded(cfg, target, exchange=SimulatedExchange(3))
    assert all(np.array_equal(a, b) for a, b in zip(got_h, ref_h))
    e1 = np.array([e for _, e in rep.error_trace])
    e0 = np.array([e for _, e in ref.error_trace])
    assert np.max(np.abs(e1 - e0) / e0) < 1e-12


@pytest.mark.parametrize("h,w,kind,levels,mask", [(12, 20, "fourier", 2, False), (10, 14, "fresnel", 4, True)])
def test_sa_any_shape_decisions_match_oracle(h, w, kind, levels, mask):
    """SA on a non-power-of-two plane (DFT tables indexed modulo H, W; packed
    element positions): every accept/reject decision equals the oracle's."""
    from paper_2006_10509_b200.search import sa_call

    cfg = _cfg(h, w, kind, levels, mask)
    cfg.algorithm, cfg.proposals = "sa", 3000
    target = _target(h, w)
    ref_holo, ref = O.sa(cfg, target, None, log_limit=3000)
    with precision("fp64"):
        holo, rep = sa_call(cfg, target, None, None, None, None, log_cap=3000)
    pix, lev, acc = rep.decisions
    want = np.array(ref.log)
    assert np.array_equal(pix, want[:, 0].astype(np.int64))
    assert np.array_equal(lev, want[:, 1].astype(np.int32))
    assert np.array_equal(acc.astype(bool), want[:, 2].astype(bool))
    assert np.array_equal(holo, ref_holo)
    assert abs(rep.final_error - ref.final_error) / ref.final_error < 1e-9


@pytest.mark.parametrize("order", ["raster", "random"])
def test_dbs_any_shape_matches_oracle(order):
    cfg = _cfg(9, 14, "fresnel", 4, True)
    cfg.algorithm, cfg.max_passes, cfg.scan_order = "dbs", 3, order
    target = _target(9, 14)
    ref_holo, ref = O.dbs(cfg, target)
    holo, rep = A.run_dbs(cfg, target)
    assert np.array_equal(holo, ref_holo)
    assert abs(rep.final_error - ref.final_error) / ref.final_error < 1e-9
    assert rep.iterations_executed == ref.iterations_executed
