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
