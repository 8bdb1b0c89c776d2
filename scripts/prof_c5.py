"""Driver for ncu captures of one C5 hologram (4096^2 Fourier PhaseOnly(8), fp32 fast passes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.workloads import batched_target

it = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = bench.make_cfg(1, n=4096, kind="fourier", iterations=it)
plan = GenerationPlan(cfg, (4096, 4096), precision=_native.FP32, device=0)
plan.set_target(batched_target(4096, 1))
rep, _ = plan.gs(cfg=cfg)
print("device_ms", rep.device_ms, "per iteration", rep.device_ms / it)
