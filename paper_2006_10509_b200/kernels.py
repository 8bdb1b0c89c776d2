"""Incremental-update kernels — drop-in for ``cghkit.kernels`` (kernels/__init__.py).

Same three functions and contract as the reference's compiled core
(``_core.pyx:20-83``), evaluated on the GPU in float64 with a fixed-order
reduction. ``BACKEND`` is ``"cuda"``; ``available_backends()`` lists only
the CUDA module (there is no CPU fallback in this package).

The runners do not call these per proposal — ``run_sa``/``run_dbs`` fuse the
same arithmetic into one persistent kernel — they exist so callers of the
reference's kernel seam keep working.
"""

from __future__ import annotations

import ctypes
import sys

import numpy as np

from . import _native
from .runtime import current_device

BACKEND = "cuda"


def _args(replay_m, target_m, row_tw, col_tw, mu, mv):
    r = np.ascontiguousarray(replay_m, dtype=np.complex128)
    t = None if target_m is None else np.ascontiguousarray(target_m, dtype=np.float64)
    rt = np.ascontiguousarray(row_tw, dtype=np.complex128)
    ct = np.ascontiguousarray(col_tw, dtype=np.complex128)
    m = np.ascontiguousarray(mu, dtype=np.int32)
    v = np.ascontiguousarray(mv, dtype=np.int32)
    return r, t, rt, ct, m, v


def delta_error(replay_m, target_m, row_tw, col_tw, mu, mv, delta):
    """sum over samples of (|R + delta w| - t)^2 - (|R| - t)^2 (_core.pyx:20-34)."""
    lib = _native.library()
    _native.require_device()
    r, t, rt, ct, m, v = _args(replay_m, target_m, row_tw, col_tw, mu, mv)
    d = complex(delta)
    out = ctypes.c_double(0.0)
    _native.check(lib.cgh_delta_error(current_device(), _native.ptr(r), _native.ptr(t), _native.ptr(rt), _native.ptr(ct),
                                      _native.ptr(m), _native.ptr(v), r.size, rt.size, ct.size, d.real, d.imag,
                                      ctypes.byref(out)))
    return float(out.value)


def commit_update(replay_m, row_tw, col_tw, mu, mv, delta):
    """replay_m += delta * row_tw[mu] * col_tw[mv], in place (_core.pyx:37-44)."""
    if not (isinstance(replay_m, np.ndarray) and replay_m.dtype == np.complex128 and replay_m.flags.c_contiguous):
        raise TypeError("replay_m must be a C-contiguous complex128 array (updated in place)")
    lib = _native.library()
    _native.require_device()
    _, _, rt, ct, m, v = _args(replay_m, None, row_tw, col_tw, mu, mv)
    d = complex(delta)
    _native.check(lib.cgh_commit_update(current_device(), _native.ptr(replay_m), _native.ptr(rt), _native.ptr(ct),
                                        _native.ptr(m), _native.ptr(v), replay_m.size, rt.size, ct.size, d.real,
                                        d.imag))


def best_delta(replay_m, target_m, row_tw, col_tw, mu, mv, deltas):
    """(index, change) of the best improving delta, (-1, 0.0) if none (_core.pyx:47-83)."""
    lib = _native.library()
    _native.require_device()
    r, t, rt, ct, m, v = _args(replay_m, target_m, row_tw, col_tw, mu, mv)
    dl = np.ascontiguousarray(deltas, dtype=np.complex128)
    bi = ctypes.c_int64(-1)
    bc = ctypes.c_double(0.0)
    _native.check(lib.cgh_best_delta(current_device(), _native.ptr(r), _native.ptr(t), _native.ptr(rt), _native.ptr(ct),
                                     _native.ptr(m), _native.ptr(v), r.size, rt.size, ct.size, _native.ptr(dl),
                                     dl.size, ctypes.byref(bi), ctypes.byref(bc)))
    return int(bi.value), float(bc.value)


def available_backends():
    """Name -> module for every backend (kernels/__init__.py:47-56): CUDA only."""
    return {"cuda": sys.modules[__name__]}
