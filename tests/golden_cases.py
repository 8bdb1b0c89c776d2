"""Rebuild the configs/inputs of tests/golden/manifest.json cases for either the
drop-in (paper_2006_10509_b200) or the oracle (duck-typed parameter objects)."""

from __future__ import annotations

import json
import os

import numpy as np

from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.image import rect_mask
from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
from paper_2006_10509_b200.slm import AmplitudeOnly, MultiAmp, PhaseOnly, SlmSpec
from paper_2006_10509_b200.workloads import aperture_beam, gaussian_beam, natural_target, square_target

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


def load_arrays(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def scheme_from(desc):
    if desc["kind"] == "phase":
        return PhaseOnly(desc["levels"], desc["offset"])
    if desc["kind"] == "amplitude":
        return AmplitudeOnly(desc["levels"])
    return MultiAmp(tuple(complex(a, b) for a, b in desc["states"]))


def build(rec):
    """(cfg, target, illumination) for a manifest record."""
    h, w = rec["height"], rec["width"]
    kind = rec["target"]
    if kind == "natural":
        target = natural_target(w, h) if h != w else natural_target(w)
    elif kind == "square":
        target = square_target(w)
    elif kind == "rect128x64":
        target = natural_target(128, 64)
    elif kind == "delta2":
        target = np.zeros((2, 2), complex)
        target[1, 1] = 1.0
    else:
        raise ValueError(kind)
    p = rec["propagation"]
    prop = PropagationSpec(p["kind"], p["wavelength"], p["distance"], p["pitch_x"], p["pitch_y"])
    mask = rect_mask(w, h, [tuple(r) for r in rec["mask_rects"]])
    params = dict(rec["params"])
    cfg = A.AlgorithmConfig(algorithm=rec["algorithm"], slm=SlmSpec(w, h, scheme_from(rec["scheme"])),
                            propagation=prop, metric=MetricSpec(mask, rec["rescale"]), **params)
    illum = {"beam": gaussian_beam, "aperture": aperture_beam}.get(rec["illumination"])
    return cfg, target, None if illum is None else illum(h, w)
