"""Where the end-to-end run_gs time goes (C3): set_target (upload + prep,
complex128 path and amplitude-only path), device GS, index download, host
expansion; and the run_gs call itself."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2006_10509_b200 import _native, algorithms as A
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.runtime import precision
from paper_2006_10509_b200.slm import states
from paper_2006_10509_b200.workloads import natural_target
n = 2048
cfg = bench.make_cfg(1, n=n, iterations=200)
t = natural_target(n)
print("host cores", len(os.sched_getaffinity(0)), flush=True)
with precision("fp32"):
    for _ in range(2): A.run_gs(cfg, t)
    ts = []
    for _ in range(15):
        t0 = time.perf_counter(); A.run_gs(cfg, t); ts.append(time.perf_counter() - t0)
    print(f"run_gs: min {1000*np.min(ts):.2f} median {1000*np.median(ts):.2f} max {1000*np.max(ts):.2f} ms", flush=True)
plan = GenerationPlan(cfg, (n, n), precision=_native.FP32, device=0)
table = states(cfg.slm.scheme)
for amp in (False, True):
    for _ in range(2):
        plan.set_target(t, amplitude_only=amp); plan.gs(); plan.download_indices(1)
    for _ in range(3):
        t0 = time.perf_counter(); plan.set_target(t, amplitude_only=amp); t1 = time.perf_counter()
        rep, _ = plan.gs(); t2 = time.perf_counter()
        idx = plan.download_indices(1)[0]; t3 = time.perf_counter()
        out = _native.expand_states(idx, table); t4 = time.perf_counter()
        print(f"amp_only={amp}: set_target {1000*(t1-t0):.2f}  gs {1000*(t2-t1):.2f} (device {rep.device_ms:.2f})  "
              f"download {1000*(t3-t2):.2f}  expand {1000*(t4-t3):.2f} ms", flush=True)

# run_gs's own sequence (prefaulted output), timed per step
from paper_2006_10509_b200.algorithms import _cached_plan, RANDOM_PHASE
with precision("fp32"):
    for rep_i in range(6):
        t0 = time.perf_counter()
        p2 = _cached_plan(cfg, t.shape)
        p2.set_target(t, None, cfg=cfg, amplitude_only=True); t1 = time.perf_counter()
        out = _native.PrefaultedArrays(t.shape); t2 = time.perf_counter()
        rep, _ = p2.gs(cfg=cfg); t3 = time.perf_counter()
        idx = p2.download_indices(1)[0]; t4 = time.perf_counter()
        o = out.take()[0]; t5 = time.perf_counter()
        holo = _native.expand_states(idx, table, out=o); t6 = time.perf_counter()
        print(f"run_gs steps: set_target {1000*(t1-t0):.2f} alloc {1000*(t2-t1):.2f} gs {1000*(t3-t2):.2f} "
              f"download {1000*(t4-t3):.2f} take {1000*(t5-t4):.2f} expand {1000*(t6-t5):.2f} total {1000*(t6-t0):.2f}",
              flush=True)
