"""SA at one plane size (binary Fourier, seed 3, auto T0 unless a third
argument gives T0): proposals per second."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.slm import SlmSpec, binary_phase
from paper_2006_10509_b200.workloads import natural_target

n = int(sys.argv[1])
props = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
cfg = bench.make_cfg(3, n=n, kind="fourier", algorithm="sa")
cfg.slm = SlmSpec(n, n, binary_phase())
if len(sys.argv) > 3:
    cfg.initial_temperature = float(sys.argv[3])
p = GenerationPlan(cfg, (n, n), precision=_native.FP64, device=0)
p.set_target(natural_target(n))
r, _ = p.sa(proposals=props)
print(f"n={n} SA {props}: {r.device_ms:.2f} ms, final {r.final_error:.10f}", flush=True)
