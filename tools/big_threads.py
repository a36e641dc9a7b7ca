import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0); s.set_option(OPT_ENGINE, 8)
cases = [("c2", W.CONFIGS["c2"].make()), ("c4", W.CONFIGS["c4"].make()),
         ("u2048", np.random.default_rng(1).integers(0, 10**6, (2048, 2048)).astype(np.int32)),
         ("g3072", W.geometric(3072, 1e6, seed=3072))]
out = [os.environ.get("KMB_BIG_THREADS", "1024")]
for name, c in cases:
    n = c.shape[0]; dc = torch.from_numpy(np.ascontiguousarray(c)).cuda()
    r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
    ts = [s.solve_into(dc, n, n, 1, r2c, u, v, tot).seconds for _ in range(2)]
    out.append(f"{name} {min(ts)*1e3:.2f}")
print("  ".join(out), flush=True)
