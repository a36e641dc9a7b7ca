import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
for key in ["c1"]:
    c = W.CONFIGS[key].make(); n = c.shape[0]
    ref = O.ref_solve_batched_km(c)
    for eng in (1, 3, 4, 5):
        s.set_option(OPT_ENGINE, eng)
        ts = []
        for _ in range(5):
            r = s.solve(c, 1); ts.append(r.stats["seconds"])
        print(key, "engine", eng, f"{min(ts)*1e3:.3f} ms", r.total_cost == ref.total_cost and np.array_equal(r.u, ref.u), flush=True)
# random sizes 129..256 parity on warp engines
rng = np.random.default_rng(9); bad = 0
for t in range(30):
    n = int(rng.integers(129, 257)); c = rng.integers(0, 5000, size=(n, n)).astype(np.int32)
    ref = O.ref_solve_batched_km(c)
    for eng in (3, 4):
        s.set_option(OPT_ENGINE, eng); r = s.solve(c, 1)
        bad += not (r.total_cost == ref.total_cost and np.array_equal(r.u, ref.u) and np.array_equal(r.v, ref.v))
print("warp engines n in 129..256 bad =", bad)
