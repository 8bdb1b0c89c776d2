"""Warp-line OSPR (2048^2 fp32, one persistent launch, CGHB200_WL_OSPR=1) vs
the batched fast path: per-frame index mismatches, trace, efficiency, device
time; binary Fourier (bench config) and 8-level Fresnel with a beam."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.slm import SlmSpec, binary_phase, PhaseOnly
from paper_2006_10509_b200.workloads import natural_target, aperture_beam

n = 2048
S = int(sys.argv[1]) if len(sys.argv) > 1 else 24


def run(cfg, beam, env):
    if not env:
        os.environ["CGHB200_WL_OSPR"] = "1"
    try:
        p = GenerationPlan(cfg, (n, n), precision=_native.FP32, device=0)
        p.set_target(natural_target(n), beam, cfg=cfg)
        p.ospr(); p.ospr()
        r, (tk, tv) = p.ospr()
        idx = p.download_indices(S)
        out = (idx.copy(), tv[:S].copy(), r.efficiency, r.device_ms)
        p.close()
        return out
    finally:
        os.environ.pop("CGHB200_WL_OSPR", None)


for name, kind, scheme, beam in (("binary fourier", "fourier", binary_phase(), None),
                                 ("8-level fresnel + beam", "fresnel", PhaseOnly(8), aperture_beam(n, n))):
    cfg = bench.make_cfg(1, n=n, kind=kind, algorithm="ospr", subframes=S)
    cfg.slm = SlmSpec(n, n, scheme)
    i1, t1, e1, ms1 = run(cfg, beam, False)
    i0, t0, e0, ms0 = run(cfg, beam, True)
    mism = [int(np.sum(a != b)) for a, b in zip(i1, i0)]
    print(f"{name}: wl {ms1:.3f} ms vs fast {ms0:.3f} ms; index mismatches per frame {mism}; "
          f"trace max rel {np.max(np.abs(t1 - t0) / t0):.2e}; eff {e1:.6f} vs {e0:.6f}", flush=True)
