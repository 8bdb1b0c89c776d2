"""Golden outputs of the reference's image.render (image.py:63-102) for a few
fields and view keys; run in the container that has /root/reference, the npz
is committed (tests/test_render.py, tests/test_gpu_render.py read it)."""
import itertools
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from cghkit import image as I  # noqa: E402

rng = np.random.default_rng(11)
fields = {
    "rand": rng.normal(size=(32, 64)) + 1j * rng.normal(size=(32, 64)),
    "phase": np.exp(1j * rng.uniform(-np.pi, np.pi, size=(64, 64))),
    "const": np.full((8, 8), 2.0 + 0j),
}
out = {}
for (fname, f), tr, view, cmap, scale in itertools.product(fields.items(), I.TRANSFORMS, I.VIEWS,
                                                            ("gray", "viridis"), I.SCALES):
    if fname == "const" and tr != "none":
        continue
    key = I.ViewKey(tr, view, cmap, scale)
    out[f"{fname}|{tr}|{view}|{cmap}|{scale}"] = I.render(f, key)
for fname, f in fields.items():
    out[f"field|{fname}"] = f
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "render_golden.npz")
np.savez_compressed(path, **out)
print(path, len(out))
