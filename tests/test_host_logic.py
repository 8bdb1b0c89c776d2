"""Host-side contract of the drop-in (CPU): parameter objects, validation order
and exception classes mirror the reference (algorithms.py:97-137,
propagation.py:48-55, slm.py:18-79, image.py:157-169)."""

import numpy as np
import pytest

from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200 import errors
from paper_2006_10509_b200.image import rect_mask
from paper_2006_10509_b200.propagation import FRESNEL, MetricSpec, PropagationSpec, fresnel_prefactor
from paper_2006_10509_b200.slm import AmplitudeOnly, MultiAmp, PhaseOnly, SlmSpec, binary_phase, states


def cfg(alg="gs", n=8, **kw):
    d = dict(algorithm=alg, slm=SlmSpec(n, n, binary_phase()), propagation=PropagationSpec(),
             metric=MetricSpec(rect_mask(n, n)), seed=7)
    d.update(kw)
    return A.AlgorithmConfig(**d)


@pytest.mark.parametrize("runner", ["gs", "sa", "dbs", "ospr"])
def test_dimension_mismatch_first(runner):
    with pytest.raises(errors.DimensionMismatchError):
        A.RUNNERS[runner](cfg(runner, 16), np.ones((8, 8), complex))
    with pytest.raises(errors.DimensionMismatchError):
        A.RUNNERS[runner](cfg(runner, 8), np.ones((8, 8), complex), illumination=np.ones((4, 4)))


@pytest.mark.parametrize("runner", ["gs", "sa", "dbs"])
def test_bad_init_mode_is_value_error(runner):
    with pytest.raises(ValueError):
        A.RUNNERS[runner](cfg(runner, init_mode="sideways"), np.ones((8, 8), complex))


@pytest.mark.parametrize("runner", ["gs", "sa", "dbs", "ospr"])
def test_invalid_spec(runner):
    for spec in (PropagationSpec(FRESNEL, distance=0.0), PropagationSpec("sideways"),
                 PropagationSpec(FRESNEL, wavelength=-1.0)):
        with pytest.raises(errors.InvalidSpecError):
            A.RUNNERS[runner](cfg(runner, propagation=spec), np.ones((8, 8), complex))


def test_mask_shape_mismatch():
    c = cfg(metric=MetricSpec(rect_mask(4, 4)))
    with pytest.raises(errors.DimensionMismatchError):
        A.run_gs(c, np.ones((8, 8), complex))


def test_states_bitwise_reference_expression():
    # slm.py:71-79
    for s in (PhaseOnly(2), PhaseOnly(7, 0.3), PhaseOnly(256)):
        k = np.arange(s.levels)
        assert np.array_equal(states(s), np.exp(1j * (s.phase_offset + 2.0 * np.pi * k / s.levels)))
    assert np.array_equal(states(AmplitudeOnly(5)), np.array([0, 0.25, 0.5, 0.75, 1.0], complex))
    assert np.array_equal(states(MultiAmp((0.2 + 0.1j, -0.5))), np.array([0.2 + 0.1j, -0.5]))
    assert binary_phase() == PhaseOnly(2, 0.0)


def test_scheme_validation():
    with pytest.raises(ValueError):
        PhaseOnly(1)
    with pytest.raises(ValueError):
        AmplitudeOnly(1)
    with pytest.raises(ValueError):
        MultiAmp((1.0,))
    with pytest.raises(ValueError):
        MultiAmp((1.0, np.inf))


def test_rect_mask():
    assert rect_mask(4, 3).shape == (3, 4) and rect_mask(4, 3).all()
    m = rect_mask(8, 8, [(1, 2, 3, 4)])
    assert m.sum() == 12 and m[2, 1] and not m[1, 1]
    with pytest.raises(errors.OutOfBoundsError):
        rect_mask(8, 8, [(6, 0, 4, 1)])


def test_fresnel_prefactor_separable_and_unit_modulus():
    spec = PropagationSpec(FRESNEL, distance=0.1)
    q = fresnel_prefactor((9, 7), spec)
    assert np.allclose(np.abs(q), 1.0, atol=1e-14)
    # the CUDA path multiplies a row factor by a column factor
    m = np.arange(9) - 4.5
    n = np.arange(7) - 3.5
    qr = np.exp(1j * np.pi * m * m * spec.pitch_y**2 / (spec.wavelength * spec.distance))
    qc = np.exp(1j * np.pi * n * n * spec.pitch_x**2 / (spec.wavelength * spec.distance))
    assert np.max(np.abs(np.outer(qr, qc) - q)) < 1e-12


def test_reference_objects_are_accepted_by_duck_typing():
    from types import SimpleNamespace

    from paper_2006_10509_b200.slm import scheme_kind

    assert scheme_kind(SimpleNamespace(levels=4, phase_offset=0.0)) == 0
    assert scheme_kind(SimpleNamespace(levels=4)) == 1
    assert scheme_kind(SimpleNamespace(state_values=(0, 1))) == 2
