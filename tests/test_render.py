"""Viewer/export rendering (cghkit/image.py:63-102) vs the reference's own
outputs (tests/golden/render_golden.npz, tests/golden/make_render_golden.py):
byte-identical for every view/colormap/scale without a transform."""

import os

import numpy as np
import pytest

from paper_2006_10509_b200.errors import NonFiniteError
from paper_2006_10509_b200.image import ViewKey, render

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "render_golden.npz"))
KEYS = sorted(k for k in G.files if not k.startswith("field|") and k.split("|")[1] == "none")


@pytest.mark.parametrize("name", KEYS)
def test_render_without_transform_is_byte_identical(name):
    fname, tr, view, cmap, scale = name.split("|")
    got = render(G[f"field|{fname}"], ViewKey(tr, view, cmap, scale))
    assert got.dtype == np.uint8 and np.array_equal(got, G[name])


def test_view_key_validation_and_nonfinite():
    with pytest.raises(ValueError):
        ViewKey(view="bogus")
    with pytest.raises(NonFiniteError):
        render(np.array([[np.nan + 0j]]), ViewKey())
