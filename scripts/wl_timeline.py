"""Stage timeline of the warp-line 2048^2 passes (CGHB200_WL_STAMPS): per
stage boundary, min / median / max over all warps of the global timer
relative to the earliest kernel entry, plus per-warp SM-clock stage durations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CGHB200_WL_STAMPS"] = "1"
import numpy as np
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.workloads import natural_target
n = 2048
cfg = bench.make_cfg(1, n=n, iterations=int(sys.argv[1]) if len(sys.argv) > 1 else 20)
plan = GenerationPlan(cfg, (n, n), precision=_native.FP32, device=0)
plan.set_target(natural_target(n))
for _ in range(3): plan.gs()
plan.profile(True); plan.gs(); passes = plan.profile(False)
print({k: round(1000 * v[0] / max(1, v[1]), 2) for k, v in passes.items()})
per = 1024 * 16 * 8 * 2
buf = np.zeros(2 * per, np.int64)
_native.check(plan.lib.cgh_debug_wl_stamps(plan.handle, _native.ptr(buf), buf.size))
names = ["entry", "pdl_wait", "stageA", "barA", "stageB", "stageC", "stageB2", "stageA2"]
for pas, nm in ((0, "ROW"), (1, "COL")):
    s = buf[pas * per:(pas + 1) * per].reshape(1024, 16, 8, 2)[:148]
    g = s[..., 0].astype(np.float64); c = s[..., 1].astype(np.float64)
    t0 = g[:, :, 0].min()
    print(f"{nm}: global timer (us after first entry), min / median / max over warps")
    for m in range(8):
        v = (g[:, :, m] - t0) / 1000
        print(f"   {names[m]:9s} {v.min():7.2f} {np.median(v):7.2f} {v.max():7.2f}")
    print(f"{nm}: per-warp stage durations (SM clocks / 1.92 GHz, us): median / max")
    for m in range(1, 8):
        d = (c[:, :, m] - c[:, :, m - 1]) / 1920
        print(f"   {names[m-1]:9s}->{names[m]:9s} {np.median(d):7.2f} {d.max():7.2f}")

# where the slowest warps are: end of stage A' per warp, by warp slot and CTA
for pas, nm in ((0, "ROW"), (1, "COL")):
    s = buf[pas * per:(pas + 1) * per].reshape(1024, 16, 8, 2)[:148]
    g = s[..., 0].astype(np.float64)
    t0 = g[:, :, 0][g[:, :, 0] > 0].min()
    end = (g[:, :, 7] - t0) / 1000
    start = (g[:, :, 1] - t0) / 1000
    valid = g[:, :, 7] > 0
    print(f"{nm}: end of pass by warp slot (median over CTAs):", np.round([np.median(end[:, w][valid[:, w]]) for w in range(16)], 2))
    ce = np.where(valid, end, 0).max(axis=1)
    print(f"{nm}: per-CTA end: min {ce.min():.2f} median {np.median(ce):.2f} max {ce.max():.2f}; slowest CTAs", np.argsort(ce)[-8:], np.round(np.sort(ce)[-8:], 2))
    print(f"{nm}: per-CTA start (pdl_wait) max {start.max():.2f}")
    d = (s[..., 1] - np.roll(s[..., 1], 1, axis=2)) / 1920.0
    for m, nmm in ((2, "A"), (4, "B"), (5, "C"), (6, "B'"), (7, "A'")):
        dm = d[:, :, m] if m != 4 else (s[:, :, 4, 1] - s[:, :, 3, 1]) / 1920.0
        if m == 2: dm = (s[:, :, 2, 1] - s[:, :, 1, 1]) / 1920.0
        dm = np.where(valid, dm, np.nan)
        print(f"   stage {nmm:3s} per-CTA median of warps: min {np.nanmin(np.nanmedian(dm,1)):.2f} max {np.nanmax(np.nanmedian(dm,1)):.2f}; quads {np.nanmedian(dm[:, :12]):.2f} pair {np.nanmedian(dm[:, 12:]):.2f}")
