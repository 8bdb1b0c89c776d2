"""Deterministic synthetic inputs for the BASELINE configs (host-side numpy).

Input generation only — not part of the compute path. The target follows
SURVEY.md §8(d): the reference acceptance suite's ``natural_target``
(``tests/test_acceptance.py:58-63``) scaled from 64 px to N px.
"""

from __future__ import annotations

import numpy as np


def natural_target(n, m=None, dx=0.0, dy=0.0):
    """Smooth two-blob target with a weak texture, amplitude in [0, 1].

    ``(dx, dy)`` shifts the blob centres by a fraction of the size (batched
    targets of config C5 use per-target offsets).
    """
    m = n if m is None else m
    out = np.empty((m, n), np.complex128)
    rows = max(1, (1 << 22) // n)   # same per-pixel formula, evaluated in row chunks (16384^2 planes)
    for a in range(0, m, rows):
        y, x = np.mgrid[a:min(m, a + rows), 0:n].astype(np.float64)
        sx, sy = n / 64.0, m / 64.0
        img = 0.3 + 0.4 * np.exp(-(((x - (20 + 64 * dx) * sx) / sx) ** 2 + ((y - (24 + 64 * dy) * sy) / sy) ** 2) / 120.0)
        img += 0.5 * np.exp(-(((x - (44 + 64 * dx) * sx) / sx) ** 2 + ((y - (40 + 64 * dy) * sy) / sy) ** 2) / 200.0)
        img += 0.15 * np.sin(x / (6.0 * sx)) * np.cos(y / (9.0 * sy))
        out[a:a + rows] = np.clip(img, 0.0, 1.0)
    return out


def batched_target(n, target_id):
    """Target ``target_id`` (1-based) of the C5 batch: per-target centre offsets
    drawn from ``default_rng(target_id)``."""
    off = np.random.default_rng(target_id).uniform(-0.1, 0.1, size=2)
    return natural_target(n, dx=float(off[0]), dy=float(off[1]))


def square_target(size, lo=0.05, hi=1.0):
    """Centred bright square (reference test fixture shape)."""
    t = np.full((size, size), lo)
    q = size // 4
    t[q : size - q, q : size - q] = hi
    return t.astype(np.complex128)


def gaussian_beam(h, w, width=0.35):
    """Smooth illumination profile (complex, zero phase)."""
    y, x = np.mgrid[0:h, 0:w].astype(np.float64)
    r2 = ((x - w / 2) / (width * w)) ** 2 + ((y - h / 2) / (width * h)) ** 2
    return np.exp(-r2).astype(np.complex128)


def aperture_beam(h, w, width=0.35, radius=0.4):
    """Gaussian illumination cut by a circular aperture: exact zeros outside
    radius * min(h, w) (exercises the zero-amplitude projection, where the
    reference's complex multiply beam * exp(i angle) yields signed zeros)."""
    y, x = np.mgrid[0:h, 0:w].astype(np.float64)
    beam = gaussian_beam(h, w, width)
    out = ((x - w / 2) ** 2 + (y - h / 2) ** 2) > (radius * min(h, w)) ** 2
    beam[out] = 0.0
    return beam
