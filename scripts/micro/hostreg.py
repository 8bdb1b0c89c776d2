"""Micro: H2D of a 64 MiB pageable numpy buffer — cudaHostRegister + DMA vs driver pageable copy."""
import ctypes, time
import numpy as np, torch
rt = ctypes.CDLL("libcudart.so.12") if False else None
cudart = torch.cuda.cudart()
n = 2048 * 2048
d = torch.empty(n * 16, dtype=torch.uint8, device="cuda")
for rep in range(4):
    a = np.random.default_rng(rep).standard_normal(2 * n)   # fresh pageable buffer (as run_gs sees it)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(torch.from_numpy(a.view(np.uint8)), non_blocking=False)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ptr = a.ctypes.data
    r = cudart.cudaHostRegister(ptr, a.nbytes, 8)   # cudaHostRegisterReadOnly
    t2 = time.perf_counter()
    d.copy_(torch.from_numpy(a.view(np.uint8)), non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    cudart.cudaHostUnregister(ptr)
    t4 = time.perf_counter()
    print(f"pageable {1e3*(t1-t0):.2f} ms | register {1e3*(t2-t1):.2f} (rc {r}) dma {1e3*(t3-t2):.2f} unregister {1e3*(t4-t3):.2f} total {1e3*(t4-t1):.2f} ms", flush=True)
