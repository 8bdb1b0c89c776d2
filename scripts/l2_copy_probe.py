"""L2-resident streaming bandwidth on this GPU: device copies of a 32 MB plane
(read + write 64 MB), timed with CUDA events; also 256 MB (HBM)."""
import torch
for mb in (32, 256):
    a = torch.empty(mb * 2**20 // 4, dtype=torch.float32, device="cuda"); b = torch.empty_like(a)
    a.normal_()
    for _ in range(5): b.copy_(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): b.copy_(a)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(f"copy {mb} MB: {ms*1000:.1f} us, {2*mb*2**20/ms/1e6:.0f} GB/s (read+write)")
