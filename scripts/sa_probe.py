"""SA throughput at the bench's C4 settings (1024^2 binary Fourier, seed 3,
auto T0, 20000 proposals; device_ms includes setup and the final report),
plus the per-proposal cost at smaller planes (T0 = 0.5) and the decision log
of the first proposals as a hash for A/B comparisons between kernel variants."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.slm import SlmSpec, binary_phase
from paper_2006_10509_b200.workloads import natural_target

cfg = bench.make_cfg(3, n=1024, kind="fourier", algorithm="sa")
cfg.slm = SlmSpec(1024, 1024, binary_phase())
cfg.proposals = 20000
p = GenerationPlan(cfg, (1024, 1024), precision=_native.FP64, device=0)
p.set_target(natural_target(1024))
p.sa(proposals=300)
for props in (2000, 20000, 60000):
    r, (tk, tv) = p.sa(proposals=props)
    h = hashlib.sha1(p.download_indices().tobytes()).hexdigest()[:12]
    print(f"C4 SA {props}: {r.device_ms:.2f} ms -> {r.iterations_executed / (r.device_ms / 1e3):.0f} proposals/s; "
          f"final {r.final_error:.12f}; trace[-2] {tv[r.trace_len - 2]:.12f}; idx sha {h}", flush=True)
p.close()
for n in (64, 256, 512, 1024):
    c = bench.make_cfg(3, n=n, kind="fourier", algorithm="sa")
    c.slm = SlmSpec(n, n, binary_phase())
    c.initial_temperature = 0.5
    q = GenerationPlan(c, (n, n), precision=_native.FP64, device=0)
    q.set_target(natural_target(n))
    q.sa(proposals=200)
    r1, _ = q.sa(proposals=1000)
    r2, _ = q.sa(proposals=6000)
    print(f"n={n} T0=0.5: {1e3 * (r2.device_ms - r1.device_ms) / 5000:.2f} us/proposal (difference of 6000 and 1000)",
          flush=True)
    q.close()
