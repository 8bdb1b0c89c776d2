"""Breakdown of one drop-in run_gs call at C3 (host API path)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.runtime import precision
from paper_2006_10509_b200.slm import states
from paper_2006_10509_b200.workloads import natural_target

cfg = bench.make_cfg(1)
target = natural_target(2048)
with precision("fp32"):
    A.run_gs(cfg, target)
    for _ in range(3):
        t0 = time.perf_counter()
        A.run_gs(cfg, target)
        t_all = time.perf_counter() - t0
        plan = A._cached_plan(cfg, target.shape)
        t0 = time.perf_counter(); plan.set_target(target, None, cfg=cfg); t_set = time.perf_counter() - t0
        t0 = time.perf_counter(); rep, _ = plan.gs(cfg=cfg); t_gs = time.perf_counter() - t0
        t0 = time.perf_counter(); idx = plan.download_indices(1)[0]; t_dl = time.perf_counter() - t0
        t0 = time.perf_counter(); h = _native.expand_states(idx, states(cfg.slm.scheme)); t_ex = time.perf_counter() - t0
        t0 = time.perf_counter(); m = A._mask_bytes(cfg, target); t_mask = time.perf_counter() - t0
        t0 = time.perf_counter(); c = _native.c128(target); t_c = time.perf_counter() - t0
        print(f"run_gs {t_all*1e3:.2f} ms | set_target {t_set*1e3:.2f} gs {t_gs*1e3:.2f} (device {rep.device_ms:.2f}) "
              f"download {t_dl*1e3:.2f} expand {t_ex*1e3:.2f} mask_bytes {t_mask*1e3:.2f} c128 {t_c*1e3:.2f}")
