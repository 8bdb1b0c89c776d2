"""Process-wide execution settings: working precision and CUDA device.

The reference computes in float64 throughout. The B200 path runs the GS/OSPR
passes in complex64 by default (the north-star fast mode, parity judged by
the 1e-4 field / 1e-3 NMSE tolerances) and offers complex128 as the parity
mode (bit-exact quantized outputs on non-chaotic configs). SA/DBS always keep
their incremental state in float64; standalone transforms and metrics default
to float64.

    CGHB200_PRECISION=fp32|fp64      runner precision (default fp32)
    CGHB200_DEVICE=<index>           CUDA device (default 0)

``precision("fp64")`` / ``device(1)`` are thread-local context managers.
"""

from __future__ import annotations

import contextlib
import os
import threading

from . import _native

_tls = threading.local()


def _parse_precision(p):
    p = str(p).lower()
    if p in ("fp32", "float32", "complex64", "32"):
        return _native.FP32
    if p in ("fp64", "float64", "complex128", "64"):
        return _native.FP64
    raise ValueError(f"unknown precision {p!r} (fp32|fp64)")


def runner_precision():
    p = getattr(_tls, "precision", None)
    if p is None:
        p = _parse_precision(os.environ.get("CGHB200_PRECISION", "fp32"))
    return p


def current_device():
    d = getattr(_tls, "device", None)
    if d is None:
        d = int(os.environ.get("CGHB200_DEVICE", "0"))
    return d


@contextlib.contextmanager
def precision(p):
    old = getattr(_tls, "precision", None)
    _tls.precision = _parse_precision(p)
    try:
        yield
    finally:
        _tls.precision = old


@contextlib.contextmanager
def device(index):
    old = getattr(_tls, "device", None)
    _tls.device = int(index)
    try:
        yield
    finally:
        _tls.device = old
