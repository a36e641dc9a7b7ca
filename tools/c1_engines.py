import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
c = W.CONFIGS["c1"].make(); n = c.shape[0]
dc = torch.from_numpy(c).cuda()
r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
for eng in (4, 6, 2, 3, 5, 1):
    s.set_option(OPT_ENGINE, eng)
    for seed in (1, 0):
        ts = [s.solve_into(dc, n, n, seed, r2c, u, v, tot).seconds for _ in range(7)]
        print(f"c1 engine {eng} seed {seed}: {min(ts)*1e3:.3f} ms tot={int(tot[0])}", flush=True)
