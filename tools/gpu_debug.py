"""Quick GPU bring-up: small parity checks with verbose output."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE

s = Solver(0)
rng = np.random.default_rng(0)
for engine in (2, 1):
    s.set_option(OPT_ENGINE, engine)
    bad = 0
    for t in range(40):
        n = int(rng.integers(1, 100)) if engine == 1 else int(rng.integers(1, 120))
        c = rng.integers(0, 50, size=(n, n)).astype(np.int32)
        ref = O.ref_solve_batched_km(c)
        try:
            r = s.solve(c, 1)
        except Exception as e:
            print("engine", engine, "n", n, "EXC", e); bad += 1; continue
        ok = r.total_cost == ref.total_cost and np.array_equal(r.u, ref.u) and np.array_equal(r.v, ref.v)
        if not ok:
            bad += 1
            if bad < 4:
                print("engine", engine, "n", n, "cost", r.total_cost, ref.total_cost, r.stats)
    print("engine", engine, "bad", bad, flush=True)
s.set_option(OPT_ENGINE, 0)
for key in ("c1", "c2"):
    c = W.CONFIGS[key].make()
    ref = O.ref_solve_batched_km(c)
    for it in range(3):
        r = s.solve(c, 1)
    print(key, r.total_cost == ref.total_cost, np.array_equal(r.u, ref.u), np.array_equal(r.v, ref.v), r.stats, flush=True)
c = W.CONFIGS["c3"].make(batch=4096)
for it in range(3):
    r = s.solve_batch(c, 1)
print("c3", r.stats, "wall", r.wall_seconds, flush=True)
for t in range(4):
    ref = O.ref_solve_batched_km(c[t])
    print("  inst", t, r.total_cost[t] == ref.total_cost, np.array_equal(r.u[t], ref.u), np.array_equal(r.v[t], ref.v))
c = W.CONFIGS["c4"].make()
for it in range(2):
    r = s.solve(c, 1)
print("c4", r.stats, flush=True)
c = W.CONFIGS["c5"].make()
for it in range(2):
    r = s.solve(c, 1)
print("c5", r.stats, flush=True)
