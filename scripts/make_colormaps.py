"""Regenerate paper_2006_10509_b200/data/colormaps.npz from the reference's
colormap tables (run in the container that has /root/reference; the output is
committed, the reference is not needed at run time). The viridis table is
public-domain (CC0) data."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from cghkit import colormaps  # noqa: E402

out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2006_10509_b200", "data",
                   "colormaps.npz")
luts = {name: np.asarray(colormaps.apply_colormap(np.arange(256) / 255.0, name), np.uint8) for name in colormaps.COLORMAPS}
np.savez(out, **luts)
print(out, {k: v.shape for k, v in luts.items()})
