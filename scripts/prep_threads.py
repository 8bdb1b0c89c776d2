import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.workloads import natural_target
n = 2048
cfg = bench.make_cfg(1, n=n, iterations=200)
t = natural_target(n)
plan = GenerationPlan(cfg, (n, n), precision=_native.FP32, device=0)
for nt in (4, 8, 12, 16, 24):
    os.environ["CGHB200_PREP_THREADS"] = str(nt)
    for _ in range(2): plan.set_target(t, amplitude_only=True)
    ts = []
    for _ in range(7):
        t0 = time.perf_counter(); plan.set_target(t, amplitude_only=True); ts.append(time.perf_counter() - t0)
    print(nt, "threads:", round(1000 * np.median(ts), 2), "ms", flush=True)
