"""OSPR 2048^2 fp32 variants on the same inputs: the default batched fast
passes and the persistent warp-line loop (CGHB200_WL_OSPR=1): per-frame index
mismatches against the first, trace, device time; binary Fourier (bench
config) and 8-level Fresnel with a beam. (A warp-line K2 over the batched
row-major frames was also measured: 1.0 ms against 0.79 ms for fast_col_holo
at 24 x 2048^2, HBM-resident planes; not kept.)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.slm import SlmSpec, binary_phase, PhaseOnly
from paper_2006_10509_b200.workloads import natural_target, aperture_beam

n = 2048
S = int(sys.argv[1]) if len(sys.argv) > 1 else 24
VARIANTS = [("default", {}), ("wl loop", {"CGHB200_WL_OSPR": "1"})]


def run(cfg, beam, env):
    os.environ.update(env)
    try:
        p = GenerationPlan(cfg, (n, n), precision=_native.FP32, device=0)
        p.set_target(natural_target(n), beam, cfg=cfg)
        p.ospr(); p.ospr()
        ms = []
        for _ in range(3):
            r, (tk, tv) = p.ospr()
            ms.append(r.device_ms)
        idx = p.download_indices(S)
        out = (idx.copy(), tv[:S].copy(), r.efficiency, min(ms))
        p.close()
        return out
    finally:
        for k in env:
            os.environ.pop(k, None)


for name, kind, scheme, beam in (("binary fourier", "fourier", binary_phase(), None),
                                 ("8-level fresnel + beam", "fresnel", PhaseOnly(8), aperture_beam(n, n))):
    cfg = bench.make_cfg(1, n=n, kind=kind, algorithm="ospr", subframes=S)
    cfg.slm = SlmSpec(n, n, scheme)
    res = [(v, run(cfg, beam, env)) for v, env in VARIANTS]
    i0, t0 = res[0][1][0], res[0][1][1]
    for v, (i1, t1, e1, ms) in res:
        mism = [int(np.sum(a != b)) for a, b in zip(i1, i0)]
        print(f"{name} [{v}]: {ms:.3f} ms; mismatches vs default {sum(mism)} (max/frame {max(mism)}); "
              f"trace max rel {np.max(np.abs(t1 - t0) / t0):.2e}; eff {e1:.6f}", flush=True)
