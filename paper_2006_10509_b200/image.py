"""``rect_mask`` — the metric-mask builder the hot path consumes (image.py:157-169)."""

from __future__ import annotations

import numpy as np

from .errors import OutOfBoundsError


def rect_mask(width: int, height: int, rects=()) -> np.ndarray:
    """Boolean mask from a union of (x, y, w, h) rectangles; empty = full plane."""
    if not rects:
        return np.ones((height, width), dtype=bool)
    mask = np.zeros((height, width), dtype=bool)
    for x, y, w, h in rects:
        if x < 0 or y < 0 or w < 0 or h < 0 or x + w > width or y + h > height:
            raise OutOfBoundsError(f"rect {(x, y, w, h)} outside {width}x{height}")
        mask[y : y + h, x : x + w] = True
    return mask
