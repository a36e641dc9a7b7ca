"""Quick engine sweep: small batches through every batch engine and the
stream-ordered call, checked against the reference.  python tools/engine_sweep.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_2005_01182_b200 import Solver, KMB_SEED_BATCHED, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
c3 = W.CONFIGS["c3"].make(batch=12)
c1 = W.CONFIGS["c1"].make()
rng = np.random.default_rng(7)
cases = [("c3 x12", c3), ("c1", c1[None]), ("n=300 x3", rng.integers(0, 1000, (3, 300, 300)).astype(np.int32))]
bad = 0
for name, c in cases:
    n = c.shape[1]
    engines = ([2, 3, 4, 6] if n <= 256 else []) + [8]
    for eng in engines:
        s.set_option(OPT_ENGINE, eng)
        r = s.solve_batch(c, KMB_SEED_BATCHED)
        ok = all(r.total_cost[t] == O.ref_solve_batched_km(c[t]).total_cost for t in range(c.shape[0]))
        bad += not ok
        print(name, "engine", eng, "ok" if ok else "MISMATCH", flush=True)
s.set_option(OPT_ENGINE, 0)
d = torch.from_numpy(c3).cuda(); b = c3.shape[0]
r2c = torch.empty((b, 128), dtype=torch.int32, device="cuda"); u = torch.empty((b, 128), dtype=torch.int64, device="cuda")
v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda"); st = torch.zeros(b, dtype=torch.int32, device="cuda")
s.solve_batch_async(d, b, 128, KMB_SEED_BATCHED, r2c, u, v, tot, st)
torch.cuda.synchronize()
print("async ok" if int(st.abs().sum()) == 0 else "async STATUS", flush=True)
print("engine_sweep:", "ok" if bad == 0 else f"{bad} mismatches")
