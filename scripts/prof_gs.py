"""Small driver for ncu captures: one GS run (default 2048^2 Fresnel PhaseOnly(8), 4 iterations)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.workloads import natural_target
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
it = int(sys.argv[2]) if len(sys.argv) > 2 else 4
prec = _native.FP64 if (len(sys.argv) > 3 and sys.argv[3] == "fp64") else _native.FP32
cfg = bench.make_cfg(1, n=n, iterations=it)
plan = GenerationPlan(cfg, (n, n), precision=prec, device=0)
plan.set_target(natural_target(n))
rep, _ = plan.gs()
print("device_ms", rep.device_ms, "final", rep.final_error)
