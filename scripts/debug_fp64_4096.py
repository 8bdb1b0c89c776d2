"""Scratch check: fp64 GS at 4096^2 alone and after an fp32 fast run."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.image import rect_mask
from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
from paper_2006_10509_b200.runtime import precision
from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec
from paper_2006_10509_b200.workloads import batched_target
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
first = sys.argv[2] if len(sys.argv) > 2 else "fp64"
cfg = A.AlgorithmConfig("gs", SlmSpec(n, n, PhaseOnly(8)), PropagationSpec("fourier"), MetricSpec(rect_mask(n, n)), seed=1, iterations=2)
t = batched_target(n, 1)
for p in ([first, "fp64"] if first != "fp64" else ["fp64"]):
    try:
        with precision(p):
            h, r = A.run_gs(cfg, t)
        print(p, "ok", r.final_error)
    except Exception as e:
        print(p, "FAIL", type(e).__name__, e)
