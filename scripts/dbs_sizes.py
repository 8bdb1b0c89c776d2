"""DBS one raster pass at one plane size (binary Fourier, seed 3): device ms per pixel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.slm import SlmSpec, binary_phase
from paper_2006_10509_b200.workloads import natural_target

n = int(sys.argv[1])
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = bench.make_cfg(3, n=n, kind="fourier", algorithm="dbs")
cfg.slm = SlmSpec(n, n, binary_phase())
p = GenerationPlan(cfg, (n, n), precision=_native.FP64, device=0)
p.set_target(natural_target(n))
r, _ = p.dbs(max_passes=passes)
print(f"n={n} DBS {passes} pass(es): {r.device_ms:.2f} ms, {r.iterations_executed} passes, "
      f"{1e3 * r.device_ms / (n * n * max(1, r.iterations_executed)):.2f} us/pixel, final {r.final_error:.10f}", flush=True)
