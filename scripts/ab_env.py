"""Interleaved A/B timing of one C3 GS run (2048^2 Fresnel PhaseOnly(8), 200
iterations) under environment-variable variants, same process and device.
Usage: ab_env.py 'VAR=1,VAR2=3' '' ...  ('' = baseline)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.workloads import natural_target
variants = [dict(kv.split("=") for kv in v.split(",") if kv) for v in (sys.argv[1:] or [""])]
n = 2048
cfg = bench.make_cfg(1, n=n, iterations=200)
plan = GenerationPlan(cfg, (n, n), precision=_native.FP32, device=0)
plan.set_target(natural_target(n))
def run(env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        rep, _ = plan.gs()
        return rep.device_ms
    finally:
        for k, v in old.items():
            if v is None: os.environ.pop(k, None)
            else: os.environ[k] = v
for v in variants: run(v); run(v)
res = {i: [] for i in range(len(variants))}
for r in range(8):
    for i, v in enumerate(variants): res[i].append(run(v))
for i, v in enumerate(variants):
    ms = np.median(res[i])
    print(f"{v or 'baseline'}: {ms:.3f} ms/run  {1000*ms/200:.2f} us/iter  (min {min(res[i]):.3f})")
