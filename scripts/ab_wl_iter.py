"""wl passes vs generic: iterations 1, 2, 3 (1 = column pass only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.runtime import precision
from paper_2006_10509_b200.workloads import natural_target

def field(cfg, t, env):
    for k in env: os.environ[k] = "1"
    try:
        with precision("fp32"):
            return A.gs_field(cfg, t, None)
    finally:
        for k in env: os.environ.pop(k, None)
n = 2048
t = natural_target(n)
for kind in ("fourier", "fresnel"):
    for it in (1, 2, 3):
        cfg = bench.make_cfg(1, n=n, kind=kind, iterations=it)
        i1, f1, r1, t1 = field(cfg, t, [])
        i3, f3, r3, t3 = field(cfg, t, ["CGHB200_NO_FAST"])
        e1 = np.array([e for _, e in t1]); e3 = np.array([e for _, e in t3])
        print(kind, it, "field rel", np.linalg.norm(f1 - f3) / np.linalg.norm(f3), "trace", e1, e3, flush=True)
