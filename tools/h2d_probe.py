"""Pinned H2D / D2H bandwidth on this box (the e2e bound)."""
import torch, time
for mb in (33.5, 268.4):
    n = int(mb * 1e6 / 4)
    h = torch.empty(n, dtype=torch.int32).pin_memory(); d = torch.empty(n, dtype=torch.int32, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [d.copy_(h, non_blocking=True) for _ in range(10)]; e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    e0.record(); [h.copy_(d, non_blocking=True) for _ in range(10)]; e1.record(); torch.cuda.synchronize()
    t2 = e0.elapsed_time(e1) / 10
    print(f"{mb} MB: H2D {t:.3f} ms = {mb/t:.1f} GB/s; D2H {t2:.3f} ms = {mb/t2:.1f} GB/s")
