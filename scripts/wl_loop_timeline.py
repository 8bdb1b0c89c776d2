"""Pass begin/end (global timer) of the persistent warp-line GS loop,
iterations 0..7: per pass the earliest begin, latest begin, latest end over
CTAs (us, relative to the loop's first begin)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CGHB200_WL_STAMPS"] = "1"
import numpy as np
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.workloads import natural_target
n = 2048
cfg = bench.make_cfg(1, n=n, iterations=20)
plan = GenerationPlan(cfg, (n, n), precision=_native.FP32, device=0)
plan.set_target(natural_target(n))
for _ in range(2): plan.gs()
plan.profile(True); plan.gs(); print(plan.profile(False))
buf = np.zeros(2 * 1024 * 16 * 8 * 2, np.int64)
_native.check(plan.lib.cgh_debug_wl_stamps(plan.handle, _native.ptr(buf), buf.size))
s = buf[: 8 * 2 * 1024 * 2].reshape(8, 2, 1024, 2)[:, :, :148].astype(np.float64)
t0 = s[0, 1, :, 0].min()
for k in range(8):
    for pas, nm in ((1, "COL"), (0, "ROW")):
        b, e = (s[k, pas, :, 0] - t0) / 1000, (s[k, pas, :, 1] - t0) / 1000
        if s[k, pas, :, 0].max() == 0: continue
        print(f"it {k} {nm}: begin {b.min():7.2f}..{b.max():7.2f}  end {e.min():7.2f}..{e.max():7.2f}  body(max) {np.max(e - b):6.2f}")

# per-CTA body durations (iterations 2..7), which CTAs are slow
dur = {}
for pas, nm in ((1, "COL"), (0, "ROW")):
    d = np.array([(s[k, pas, :, 1] - s[k, pas, :, 0]) / 1000 for k in range(2, 8)])
    m = d.mean(axis=0)
    dur[nm] = m
    order = np.argsort(m)
    print(f"{nm}: body us per CTA: min {m.min():.2f} median {np.median(m):.2f} max {m.max():.2f}")
    print(f"   slowest 12 CTAs {order[-12:].tolist()}  {np.round(m[order[-12:]], 1).tolist()}")
    print(f"   fastest 6 CTAs {order[:6].tolist()}  {np.round(m[order[:6]], 1).tolist()}")
    hist = np.histogram(m, bins=8)
    print("   histogram", hist[0].tolist(), np.round(hist[1], 1).tolist())
    print("   CTAs >= 136 (no pair):", np.round(m[136:], 1).tolist())
