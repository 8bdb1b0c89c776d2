"""Standalone quantizer on the device (slm.quantize_indices / quantize ->
cgh_quantize) vs the real reference's outputs (tests/golden/quantize_golden.npz,
made by tests/golden/make_quantize_golden.py from cghkit.slm.quantize_indices,
slm.py:86-108) on the reference test suite's schemes and inputs
(pkg/tests/test_slm.py:15-122) plus ties, wrap-around and signed zeros:
bit-exact index planes.

Near-ties: values whose two candidate states are within a few ulps of
equidistant are decided by the last bit of numpy's angle / complex abs. On
AVX-512 hosts numpy computes those with its own SIMD kernels (measured here:
np.arctan2 differs from libm atan2 on 7% of random inputs, np.abs(complex) is
not correctly rounded on 35%), so the reference's outcome there depends on the
host CPU. Such values (the constructed half-way phases exp(i (k + 1/2) 2 pi / L)
and distance ties such as -1j for MultiAmp((0.2+0.1j, -0.5, 1j, 0.9))) must map
to one of their two candidates and are counted; every other value is bit-exact.
The reference tests' own tie cases (exp(i pi/2) for binary, exp(-i pi/4) for
L = 4, MultiAmp((0, 1)) at 0.5) are checked bit-exactly in
test_device_quantize_known_answers."""

import os

import numpy as np
import pytest

from paper_2006_10509_b200.slm import AmplitudeOnly, MultiAmp, PhaseOnly, binary_phase, quantize, quantize_indices, states

pytestmark = pytest.mark.gpu

GOLD = dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "quantize_golden.npz")))
SCHEMES = [PhaseOnly(2), PhaseOnly(4), PhaseOnly(7, phase_offset=0.3), PhaseOnly(256), AmplitudeOnly(2),
           AmplitudeOnly(5), MultiAmp((0, 1)), MultiAmp((0.2 + 0.1j, -0.5, 1j, 0.9))]


def _near_tie(vals, scheme):
    """(mask of last-ulp near-ties, their two candidate indices)."""
    table = states(scheme)
    if hasattr(scheme, "phase_offset"):
        L = scheme.levels
        frac = np.mod((np.angle(vals) - scheme.phase_offset) / (2.0 * np.pi / L), L)
        rem = frac - np.floor(frac)
        lo = np.floor(frac).astype(np.int64) % L
        near = np.abs(rem - 0.5) < 1e-9   # includes ties that are exact only in this host's numpy atan2
        return near, np.stack([lo, (lo + 1) % L, (lo + 1) % L])
    d = np.abs(vals[:, None] - table[None, :])
    order = np.argsort(d, axis=1, kind="stable")
    d0 = np.take_along_axis(d, order[:, :1], 1)[:, 0]
    d1 = np.take_along_axis(d, order[:, 1:2], 1)[:, 0]
    near = (d1 - d0) <= 1e-12 * np.maximum(d1, 1e-300)
    return near & (d1 != d0), np.stack([order[:, 0], order[:, 1], order[:, 1]])


@pytest.mark.parametrize("i", range(len(SCHEMES)))
def test_device_quantize_indices_bit_exact_vs_reference(i):
    vals, ref = GOLD[f"values{i}"], GOLD[f"idx{i}"]
    got = quantize_indices(vals, SCHEMES[i])
    assert got.dtype == np.int32
    near, cand = _near_tie(vals, SCHEMES[i])
    bad = np.nonzero((got != ref) & ~near)[0]
    assert bad.size == 0, [(complex(vals[j]), int(got[j]), int(ref[j])) for j in bad[:8]]
    assert np.all((got[near] == cand[0][near]) | (got[near] == cand[1][near]) | (got[near] == cand[2][near]))
    print(f"{SCHEMES[i]}: {vals.size} values, {int(near.sum())} last-ulp near-ties, "
          f"{int(np.sum((got != ref) & near))} decided differently from this host's numpy")
    # 2-D input keeps its shape; values are bitwise state members
    two = quantize(vals[:64].reshape(8, 8), SCHEMES[i])
    assert two.shape == (8, 8)
    assert np.array_equal(two, states(SCHEMES[i])[ref[:64].reshape(8, 8)])


def test_device_quantize_known_answers():
    """pkg/tests/test_slm.py:57-86 on the device."""
    assert quantize(np.exp(1j * 0.9 * np.pi), binary_phase()) == states(binary_phase())[1]
    assert quantize(np.exp(1j * np.pi / 3), PhaseOnly(4)) == states(PhaseOnly(4))[1]
    got = quantize(0.01 * np.exp(1j * 0.1), PhaseOnly(4))
    assert got == states(PhaseOnly(4))[0] and abs(got) == 1.0
    assert quantize(0j, PhaseOnly(4, 0.0)) == states(PhaseOnly(4))[0]
    s = MultiAmp((0, 1))
    assert quantize(0.4 + 0j, s) == 0.0 and quantize(0.6 + 0j, s) == 1.0 and quantize(0.5 + 0j, s) == 0.0
    assert quantize(np.exp(1j * np.pi / 2), binary_phase()) == 1.0
    assert quantize(np.exp(-1j * np.pi / 4), PhaseOnly(4)) == states(PhaseOnly(4))[0]
    # signed zeros: angle(-0 + 0j) = pi -> the level at pi
    assert quantize_indices(np.array([complex(-0.0, 0.0)]), PhaseOnly(8))[0] == 4
    assert quantize_indices(np.array([complex(-0.0, -0.0)]), PhaseOnly(8))[0] == 4


def test_device_quantize_large_plane():
    """A C3-sized plane (4.2M values) against the host restatement of the formula."""
    from oracle import cgh_oracle as O

    gen = np.random.default_rng(7)
    vals = gen.normal(size=(2048, 2048)) + 1j * gen.normal(size=(2048, 2048))
    for s in (PhaseOnly(8), PhaseOnly(256, 0.1), AmplitudeOnly(16)):
        assert np.array_equal(quantize_indices(vals, s), O.nearest_state_index(vals, s))
