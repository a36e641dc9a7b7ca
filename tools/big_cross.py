"""Single-CTA (8) vs cluster (5) engine by n (uniform and geometric-like costs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
rng = np.random.default_rng(1)
for n in (300, 512, 768, 1024, 1536, 2048, 3072):
    for kind in ("uniform", "geom"):
        if kind == "uniform":
            c = rng.integers(0, 10**6, (n, n)).astype(np.int32)
        else:
            c = W.geometric(n, 1e6, seed=n)
        dc = torch.from_numpy(np.ascontiguousarray(c)).cuda()
        r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
        v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
        res = []
        for eng in (5, 8):
            s.set_option(OPT_ENGINE, eng)
            ts = [s.solve_into(dc, n, n, 1, r2c, u, v, tot).seconds for _ in range(2)]
            res.append(f"e{eng} {min(ts)*1e3:.2f} ms")
        print(f"n={n} {kind}: " + "  ".join(res), flush=True)
