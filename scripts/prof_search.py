"""Timing sweep / ncu driver for the SA and DBS search kernels."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200.plan import GenerationPlan
from paper_2006_10509_b200.slm import SlmSpec, binary_phase
from paper_2006_10509_b200.workloads import natural_target
sizes = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["256", "512", "1024"])]
props = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
do_dbs = len(sys.argv) <= 3 or sys.argv[3] != "sa"
for n in sizes:
    cfg = bench.make_cfg(3, n=n, kind="fourier", algorithm="sa")
    cfg.slm = SlmSpec(n, n, binary_phase())
    cfg.initial_temperature = 0.5
    p = GenerationPlan(cfg, (n, n), precision=_native.FP64, device=0)
    p.set_target(natural_target(n))
    p.sa(proposals=200)
    r, _ = p.sa(proposals=props)
    line = f"n={n} SA {props} proposals: {r.device_ms:.2f} ms -> {1000*r.device_ms/props:.2f} us/proposal"
    if do_dbs and n <= 512:
        rd, _ = p.dbs(max_passes=1)
        line += f" | DBS 1 pass: {rd.device_ms:.2f} ms -> {1e3*rd.device_ms/(n*n):.2f} us/pixel"
    print(line, flush=True)
