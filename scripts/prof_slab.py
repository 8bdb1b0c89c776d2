"""Driver for ncu captures of the slab (C6) path: one G = 1 run of N^2 (default 16384), 2 iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200 import slab as SL
from paper_2006_10509_b200.workloads import natural_target

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
it = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = bench.make_cfg(1, n=n, kind="fourier", iterations=it)
sess = SL.SlabSession(cfg, natural_target(n), precision=_native.FP32, device=0)
sums, done, _ = sess.run()
print("errors", sess.errors(sums, done))
sess.close()
