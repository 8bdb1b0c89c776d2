import time, torch, numpy as np, ctypes, sys
sys.path.insert(0,'.')
from paper_2006_10509_b200 import _native
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.runtime import precision
import bench
from paper_2006_10509_b200.workloads import natural_target
n=2048
x=np.random.rand(n,n)+1j*np.random.rand(n,n)
pin=torch.empty(n*n*16,dtype=torch.uint8).pin_memory()
dev=torch.empty(n*n*16,dtype=torch.uint8,device='cuda')
pn=pin.numpy()
for _ in range(3):
    t0=time.perf_counter(); dev.copy_(pin,non_blocking=True); torch.cuda.synchronize(); t1=time.perf_counter()
    np.copyto(pn, x.view(np.uint8).reshape(-1)); t2=time.perf_counter()
    dev.copy_(torch.from_numpy(x.view(np.uint8).reshape(-1))); torch.cuda.synchronize(); t3=time.perf_counter()
    print(f"pinned H2D {(t1-t0)*1e3:.2f} ms  host memcpy 1 thread {(t2-t1)*1e3:.2f} ms  pageable H2D {(t3-t2)*1e3:.2f} ms")
cfg = bench.make_cfg(1)
target = natural_target(2048)
with precision("fp32"):
    A.run_gs(cfg, target)
    plan = A._cached_plan(cfg, target.shape)
    m = A._mask_bytes(cfg, target)
    lib=_native.library()
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); plan.set_target(target, None, cfg=cfg); t1=time.perf_counter()
        lib.cgh_plan_sync(plan.handle) if hasattr(plan,'handle') else None
        torch.cuda.synchronize(); t2=time.perf_counter()
        print(f"set_target call {(t1-t0)*1e3:.2f} ms, +sync {(t2-t1)*1e3:.2f}")
