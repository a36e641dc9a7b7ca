import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
cases = [("u4096", np.random.default_rng(4).integers(0, 10**6, (4096, 4096)).astype(np.int32)),
         ("g4096", W.geometric(4096, 1e6, seed=44)), ("g6144", W.geometric(6144, 1e6, seed=61)),
         ("u5120", np.random.default_rng(5).integers(0, 10**6, (5120, 5120)).astype(np.int32))]
for name, c in cases:
    n = c.shape[0]; dc = torch.from_numpy(c).cuda()
    r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
    out = []
    for eng in (1, 5, 8):
        if eng == 8 and n > 4096: continue
        s.set_option(OPT_ENGINE, eng)
        ts = [s.solve_into(dc, n, n, 1, r2c, u, v, tot).seconds for _ in range(2)]
        out.append(f"e{eng} {min(ts)*1e3:.1f}")
    print(name, "  ".join(out), flush=True)
