"""Config 4 on the cluster engine with its matrix at different device
allocations: is the allocation-placement effect (129 vs 142-144 ms) bimodal?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
s = Solver(0)
c = W.CONFIGS["c4"].make(); n = c.shape[0]
host = torch.from_numpy(c)
r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
big = torch.empty((3 << 30) // 4, dtype=torch.int32, device="cuda")  # 3 GiB arena
step = (256 << 20) // 4
for k in range(10):
    off = k * step
    view = big[off: off + n * n].view(n, n)
    view.copy_(host)
    ts = [s.solve_into(view, n, n, 1, r2c, u, v, tot).seconds for _ in range(2)]
    print(f"offset {k * 256} MiB: {min(ts) * 1e3:.1f} ms  ptr {view.data_ptr():#x}", flush=True)
