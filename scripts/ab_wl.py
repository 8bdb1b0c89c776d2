"""A/B of the warp-line 2048^2 passes against the previous fast passes and
the generic passes: field / trace agreement and device time per GS run."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2006_10509_b200 import _native, algorithms as A
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.runtime import precision
from paper_2006_10509_b200.workloads import natural_target, gaussian_beam

def field(cfg, target, illum, env):
    old = {k: os.environ.pop(k, None) for k in ("CGHB200_NO_WL", "CGHB200_NO_FAST", "CGHB200_WL_NO_LOOP")}
    for k in env: os.environ[k] = "1"
    try:
        with precision("fp32"):
            return A.gs_field(cfg, target, illum)
    finally:
        for k in env: os.environ.pop(k, None)
        for k, v in old.items():
            if v is not None: os.environ[k] = v

n = 2048
for kind, beam, gain, rescale in (("fresnel", False, 0.0, False), ("fourier", True, 0.3, True)):
    cfg = bench.make_cfg(1, n=n, kind=kind, iterations=5)
    cfg.feedback_gain = gain
    cfg.metric.rescale = rescale
    t = natural_target(n)
    il = gaussian_beam(n, n) if beam else None
    i1, f1, r1, t1 = field(cfg, t, il, [])
    i2, f2, r2, t2 = field(cfg, t, il, ["CGHB200_WL_NO_LOOP"])
    i3, f3, r3, t3 = field(cfg, t, il, ["CGHB200_NO_FAST"])
    e1 = np.array([e for _, e in t1]); e3 = np.array([e for _, e in t3])
    print(kind, "beam" if beam else "", "wl vs generic field rel", np.linalg.norm(f1 - f3) / np.linalg.norm(f3),
          "wl per-pass vs generic", np.linalg.norm(f2 - f3) / np.linalg.norm(f3),
          "trace rel", np.max(np.abs(e1 - e3) / e3), "idx mism", int(np.sum(i1 != i3)), flush=True)

cfg = bench.make_cfg(1, n=n, iterations=200)
for env in ([], ["CGHB200_WL_NO_LOOP"], ["CGHB200_NO_WL"]):
    for k in env: os.environ[k] = "1"
    plan = GenerationPlan(cfg, (n, n), precision=_native.FP32, device=0)
    plan.set_target(natural_target(n))
    for _ in range(3): plan.gs()
    ms = []
    for _ in range(10):
        rep, _ = plan.gs(); ms.append(rep.device_ms)
    plan.profile(True); plan.gs(); passes = plan.profile(False)
    print("env", env, "ms/run", np.median(ms), "us/iter", 1000 * np.median(ms) / 200,
          {k: round(1000 * v[0] / max(1, v[1]), 2) for k, v in passes.items()}, flush=True)
    plan.close()
    for k in env: os.environ.pop(k, None)
