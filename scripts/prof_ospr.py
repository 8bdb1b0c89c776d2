"""Per-pass timing of one OSPR run (default C2: 1024^2 binary, 24 subframes)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.slm import SlmSpec, binary_phase
from paper_2006_10509_b200.workloads import natural_target
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
S = int(sys.argv[2]) if len(sys.argv) > 2 else 24
cfg = bench.make_cfg(1, n=n, kind="fourier", algorithm="ospr", subframes=S)
cfg.slm = SlmSpec(n, n, binary_phase())
p = GenerationPlan(cfg, (n, n), precision=_native.FP32, device=0)
p.set_target(natural_target(n))
p.ospr()
p.profile(True)
r, _ = p.ospr()
print("device_ms", r.device_ms, p.profile(False))
