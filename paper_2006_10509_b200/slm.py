"""Modulator models and state quantization (drop-in for ``cghkit/slm.py``).

The scheme/spec dataclasses mirror ``slm.py:18-64``; ``states`` builds the
state table with the reference's own numpy expression (``slm.py:71-79``) so
values are bitwise identical and returned holograms are bitwise members of
the state set. ``quantize_indices`` runs on the GPU (``cgh_quantize``, fp64,
the closed-form / first-argmin rule of ``slm.py:86-108``).

Scheme objects are recognised by attributes, so the reference's own
``PhaseOnly``/``AmplitudeOnly``/``MultiAmp`` instances work as well.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native


@dataclass(frozen=True)
class PhaseOnly:
    """Unit-modulus states exp(i (offset + 2 pi k / levels)) (slm.py:18-31)."""

    levels: int
    phase_offset: float = 0.0

    def __post_init__(self):
        if self.levels < 2:
            raise ValueError("phase-only scheme needs at least 2 levels")


def binary_phase() -> PhaseOnly:
    """Phases 0 and pi (slm.py:28-31)."""
    return PhaseOnly(2, 0.0)


@dataclass(frozen=True)
class AmplitudeOnly:
    """Real states k / (levels - 1) (slm.py:34-42)."""

    levels: int

    def __post_init__(self):
        if self.levels < 2:
            raise ValueError("amplitude-only scheme needs at least 2 levels")


@dataclass(frozen=True)
class MultiAmp:
    """Arbitrary finite complex state set; order fixes tie-breaking (slm.py:45-55)."""

    state_values: tuple

    def __post_init__(self):
        if len(self.state_values) < 2:
            raise ValueError("multi-amp scheme needs at least 2 states")
        if not np.all(np.isfinite(np.asarray(self.state_values, dtype=np.complex128))):
            raise ValueError("multi-amp states must be finite")


@dataclass(frozen=True)
class SlmSpec:
    """Device resolution plus modulation scheme (slm.py:58-64)."""

    width: int
    height: int
    scheme: object


def _scheme_of(obj):
    return obj.scheme if hasattr(obj, "scheme") and hasattr(obj, "width") else obj


def scheme_kind(scheme):
    """C-ABI scheme code from the object's attributes."""
    scheme = _scheme_of(scheme)
    if hasattr(scheme, "state_values"):
        return _native.SCHEME_MULTI
    if hasattr(scheme, "phase_offset"):
        return _native.SCHEME_PHASE
    if hasattr(scheme, "levels"):
        return _native.SCHEME_AMPLITUDE
    raise TypeError(f"not a modulation scheme: {scheme!r}")


def states(scheme) -> np.ndarray:
    """State table as complex128 in index order (slm.py:71-79)."""
    scheme = _scheme_of(scheme)
    kind = scheme_kind(scheme)
    if kind == _native.SCHEME_PHASE:
        k = np.arange(scheme.levels)
        return np.exp(1j * (scheme.phase_offset + 2.0 * np.pi * k / scheme.levels))
    if kind == _native.SCHEME_AMPLITUDE:
        return (np.arange(scheme.levels) / (scheme.levels - 1)).astype(np.complex128)
    return np.asarray(scheme.state_values, dtype=np.complex128)


def problem_for(scheme, height, width, precision, device=0):
    """Fill a C ``cgh_problem`` for this scheme (propagation/metric set later).

    Returns (problem, keepalive) — the state array must outlive the call.
    """
    scheme = _scheme_of(scheme)
    table = np.ascontiguousarray(states(scheme), dtype=np.complex128)
    pb = _native.Problem()
    pb.height = int(height)
    pb.width = int(width)
    pb.precision = int(precision)
    pb.device = int(device)
    pb.scheme_kind = scheme_kind(scheme)
    pb.n_states = len(table)
    pb.phase_offset = float(getattr(scheme, "phase_offset", 0.0))
    pb.states = table.ctypes.data
    return pb, table


def quantize_indices(values, scheme) -> np.ndarray:
    """Index of the nearest allowed state for every value (slm.py:86-108), on the GPU."""
    scheme = _scheme_of(scheme)
    values = np.asarray(values, dtype=np.complex128)
    flat = np.ascontiguousarray(values.reshape(-1))
    out = np.empty(flat.shape[0], dtype=np.int32)
    if flat.size:
        lib = _native.library()
        _native.require_device()
        from .runtime import current_device

        pb, keep = problem_for(scheme, 1, 1, _native.FP64, current_device())
        _native.check(lib.cgh_quantize(ctypes.byref(pb), _native.ptr(flat), flat.size, _native.ptr(out)))
        del keep
    return out.reshape(values.shape)


def quantize(values, scheme):
    """Snap a field (or a single value) to the scheme's states (slm.py:111-116)."""
    scalar = np.isscalar(values) or np.asarray(values).ndim == 0
    idx = quantize_indices(values, scheme)
    snapped = states(scheme)[idx]
    return complex(snapped) if scalar else snapped
