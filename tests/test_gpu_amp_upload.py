"""The amplitude-only target upload (cgh_plan_set_target_ex flag 1: host
threads build the shifted, mask-signed fp32 amplitude, SSE2 rows with a
scalar fallback for rows holding tiny / huge / non-finite values) against the
complex128 upload whose amplitude the device computes (prep_kernel): same GS
index plane and trace, on planes that take the vectorised rows (even widths),
the scalar rows only (odd half width), and the warp-line 2048^2 path; with a
metric mask, zero pixels and a row of sub-1e-150 magnitudes."""

import numpy as np
import pytest

from paper_2006_10509_b200 import _native
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.image import rect_mask
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec

pytestmark = pytest.mark.gpu


def _target(h, w, seed):
    g = np.random.default_rng(seed)
    t = (g.random((h, w)) * np.exp(2j * np.pi * g.random((h, w)))).astype(np.complex128)
    t[g.random((h, w)) < 0.2] = 0.0                 # dark pixels
    t[h // 3] = 1e-160 * (1 + 1j)                    # squares underflow: scalar row
    return t


@pytest.mark.parametrize("h,w", [(256, 384), (130, 98), (2048, 2048)])
def test_amplitude_only_upload_matches_device_prep(h, w):
    mask = rect_mask(w, h)
    mask[: h // 8] = False                            # part of the plane outside the metric
    cfg = A.AlgorithmConfig("gs", SlmSpec(w, h, PhaseOnly(8)), PropagationSpec("fresnel", distance=0.05),
                            MetricSpec(mask), seed=5, iterations=3)
    target = _target(h, w, h + w)
    plan = GenerationPlan(cfg, (h, w), precision=_native.FP32, device=0)
    try:
        out = []
        for amp in (False, True):
            plan.set_target(target, cfg=cfg, amplitude_only=amp)
            rep, (tk, tv) = plan.gs()
            out.append((plan.download_indices(1)[0].copy(), tv[: rep.iterations_executed + 1].copy()))
        (i0, t0), (i1, t1) = out
        assert np.array_equal(i0, i1)
        assert np.max(np.abs(t1 - t0) / np.abs(t0)) < 1e-12
    finally:
        plan.close()
