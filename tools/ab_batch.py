"""A/B the per-instance engines on config 3 (and random small parity)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE

s = Solver(0)
rng = np.random.default_rng(0)
for engine in (2, 3, 4, 6):
    s.set_option(OPT_ENGINE, engine)
    bad = 0
    for t in range(60):
        n = int(rng.integers(1, 200 if engine > 2 else 120))
        c = rng.integers(0, int(rng.choice([3, 50, 10**6, 10**8])), size=(n, n)).astype(np.int32)
        ref = O.ref_solve_batched_km(c)
        for seed in (1, 0):
            if seed == 0:
                ref = O.ref_solve_km(c)
            r = s.solve(c, seed)
            if not (r.total_cost == ref.total_cost and np.array_equal(r.u, ref.u) and np.array_equal(r.v, ref.v)):
                bad += 1
                if bad < 3: print("MISMATCH engine", engine, "n", n, "seed", seed, r.total_cost, ref.total_cost, flush=True)
    print("engine", engine, "random parity bad =", bad, flush=True)
c = W.CONFIGS["c3"].make()
b, n, _ = c.shape
dc = torch.from_numpy(c).cuda()
r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
ref_tot = None
for engine in (2, 3, 4, 6):
    s.set_option(OPT_ENGINE, engine)
    ts = []
    for it in range(5):
        st = s.solve_batch_into(dc, b, n, 1, r2c, u, v, tot)
        ts.append(st.seconds)
    if ref_tot is None: ref_tot = tot.clone(); ref_u = u.clone()
    same = bool(torch.equal(tot, ref_tot)) and bool(torch.equal(u, ref_u))
    print(f"c3 engine {engine}: {min(ts)*1e3:.3f} ms  ({b/min(ts):.0f} solves/s) same={same} phases={st.phases} ds={st.dual_steps} rounds={st.rounds} rows={st.rows_scanned} inst_cycles max={st.max_instance_cycles} mean={st.sum_instance_cycles/b:.0f}", flush=True)
