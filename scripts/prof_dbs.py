import sys, os, time
sys.path.insert(0, "/root/repo")
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.slm import SlmSpec, binary_phase
from paper_2006_10509_b200.workloads import natural_target
n = int(sys.argv[1])
cfg = bench.make_cfg(3, n=n, kind="fourier", algorithm="dbs")
cfg.slm = SlmSpec(n, n, binary_phase())
p = GenerationPlan(cfg, (n, n), precision=_native.FP64, device=0)
p.set_target(natural_target(n))
t0 = time.time()
rd, _ = p.dbs(max_passes=1)
print(n, "DBS pass", rd.device_ms, "ms", 1e3 * rd.device_ms / (n * n), "us/px", time.time() - t0, flush=True)
