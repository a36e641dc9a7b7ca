import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2005_01182_b200 import Solver, KMB_SEED_BATCHED
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
rng = np.random.default_rng(3)
n = int(rng.integers(2, 300)); c = rng.integers(0, 20, size=(n, n)).astype(np.int32)
mi = O.mirror_solve_incr(c, 1)
s.set_option(OPT_ENGINE, 5)
res = [s.solve(c, KMB_SEED_BATCHED) for _ in range(6)]
print(os.environ.get("KMB_NO_DSM"), n, "phases", [r.stats["phases"] for r in res], "mirror", mi.phases, "same-as-mirror", [bool(np.array_equal(r.row_to_col, mi.row_to_col)) for r in res])
