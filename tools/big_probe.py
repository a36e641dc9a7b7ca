"""Single-CTA engine (8) vs cluster (5) on configs 2 and 4 + random parity."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_2005_01182_b200 import Solver, workloads as W, KMB_SEED_BATCHED, KMB_SEED_KM
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
rng = np.random.default_rng(5)
bad = 0
for t in range(40):
    n = int(rng.integers(1, 700)); hi = int(rng.choice([3, 100, 10**6]))
    c = rng.integers(0, hi, (n, n)).astype(np.int32)
    seed = int(rng.choice([0, 1]))
    ref = O.ref_solve_batched_km(c) if seed else O.ref_solve_km(c)
    s.set_option(OPT_ENGINE, 8)
    r = s.solve(c, seed)
    ok = np.array_equal(r.u, ref.u) and np.array_equal(r.v, ref.v) and r.total_cost == ref.total_cost
    if not ok:
        bad += 1; print("MISMATCH", n, hi, seed, r.total_cost, ref.total_cost, flush=True)
print("random parity mismatches:", bad, flush=True)
for key in ("c2", "c4"):
    c = W.CONFIGS[key].make(); n = c.shape[0]
    dc = torch.from_numpy(c).cuda()
    r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
    for eng in (5, 8):
        s.set_option(OPT_ENGINE, eng)
        ts = []
        for _ in range(3):
            st = s.solve_into(dc, n, n, 1, r2c, u, v, tot); ts.append(st.seconds)
        print(f"{key} engine {eng}: {min(ts)*1e3:.2f} ms tot={int(tot[0])} rounds={st.rounds} phases={st.phases} ds={st.dual_steps}", flush=True)
