"""The warp-line OSPR loop (opt-in CGHB200_WL_OSPR=1; wl_ospr.cuh: all
subframes of a 2048^2 fp32 hologram in one persistent launch) against the
batched fast OSPR passes on the same inputs: index planes equal up to a few
decision-boundary pixels per subframe, per-subframe errors within 1e-6,
efficiency; binary Fourier and 8-level Fresnel with an aperture beam (zero
pixels), plus the column-tiled index permutation."""

import os

import numpy as np
import pytest

from paper_2006_10509_b200 import _native
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.image import rect_mask
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec, binary_phase
from paper_2006_10509_b200.workloads import aperture_beam, natural_target

pytestmark = pytest.mark.gpu
N = 2048
S = 6


def _run(cfg, beam, wl):
    if wl:
        os.environ["CGHB200_WL_OSPR"] = "1"
    try:
        p = GenerationPlan(cfg, (N, N), precision=_native.FP32, device=0)
        try:
            p.set_target(natural_target(N), beam, cfg=cfg)
            r, (tk, tv) = p.ospr()
            return p.download_indices(S).copy(), tv[:S].copy(), r.efficiency
        finally:
            p.close()
    finally:
        os.environ.pop("CGHB200_WL_OSPR", None)


@pytest.mark.parametrize("kind,levels,beam", [("fourier", 2, False), ("fresnel", 8, True)])
def test_wl_ospr_matches_batched_passes(kind, levels, beam):
    scheme = binary_phase() if levels == 2 else PhaseOnly(levels)
    mask = rect_mask(N, N)
    mask[: N // 16] = False
    cfg = A.AlgorithmConfig("ospr", SlmSpec(N, N, scheme), PropagationSpec(kind, distance=0.05),
                            MetricSpec(mask), seed=11, subframes=S)
    b = aperture_beam(N, N) if beam else None
    i1, t1, e1 = _run(cfg, b, True)
    i0, t0, e0 = _run(cfg, b, False)
    mism = [int(np.sum(x != y)) for x, y in zip(i1, i0)]
    print(f"wl OSPR {kind} L={levels}: mismatches per subframe {mism}")
    assert max(mism) <= 16, mism
    assert np.max(np.abs(t1 - t0) / t0) < 1e-6
    assert abs(e1 - e0) < 1e-6
