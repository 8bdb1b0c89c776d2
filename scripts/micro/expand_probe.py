"""Host expansion states[idx] into a fresh vs a pre-faulted complex128 array (C3 size)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

from paper_2006_10509_b200 import _native

print("thp:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
n = 2048
idx = np.random.default_rng(0).integers(0, 8, (n, n)).astype(np.uint8)
table = np.exp(2j * np.pi * np.arange(8) / 8)
lib = _native.library()
for _ in range(4):
    t0 = time.perf_counter()
    out = _native.expand_states(idx, table)
    t1 = time.perf_counter()
    pre = np.empty((n, n), np.complex128)
    t2 = time.perf_counter()
    pre.view(np.uint8)[:, ::4096] = 0   # touch every page
    t3 = time.perf_counter()
    _native.check(lib.cgh_expand_states(_native.ptr(idx), 1, idx.size, _native.ptr(table), 8, _native.ptr(pre), 16))
    t4 = time.perf_counter()
    print(f"fresh {1e3*(t1-t0):.2f} ms | touch pages {1e3*(t3-t2):.2f} ms, expand into touched {1e3*(t4-t3):.2f} ms")
