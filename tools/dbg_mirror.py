import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2005_01182_b200 import Solver, KMB_SEED_BATCHED
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
rng = np.random.default_rng(3)
for t in range(20):
    n = int(rng.integers(2, 300))
    c = rng.integers(0, 20, size=(n, n)).astype(np.int32)
    mi = O.mirror_solve_incr(c, 1)
    ref = O.ref_solve_batched_km(c)
    for engine in [1, 5]:
        s.set_option(OPT_ENGINE, engine)
        r = s.solve(c, KMB_SEED_BATCHED)
        ok = np.array_equal(r.row_to_col, mi.row_to_col)
        duals = np.array_equal(r.u, ref.u) and np.array_equal(r.v, ref.v)
        if not ok or not duals:
            print(f"t={t} n={n} engine={engine} match_ok={ok} duals_ok={duals} tot={r.total_cost} ref={ref.total_cost} phases {r.stats['phases']} vs {mi.phases} rounds {r.stats['rounds']} vs {mi.rounds}", flush=True)
