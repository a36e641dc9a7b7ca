"""Randomised stress: engines x sizes x value ranges x seeds against the
reference (duals, total cost) and against themselves (determinism: the same
matching and round count twice).  Usage: python tools/stress.py [seconds]
(BATCH=1: random batches through every batch engine instead)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2005_01182_b200 import Solver, KMB_SEED_BATCHED, KMB_SEED_KM
from paper_2005_01182_b200.api import OPT_ENGINE
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
s = Solver(0)
rng = np.random.default_rng(int(os.environ.get("SEED", "12345")))
t0 = time.time(); cases = 0; bad = 0
while time.time() - t0 < budget:
    hi = int(rng.choice([2, 10, 1000, 10**6, 2**29 - 1]))
    if os.environ.get("BATCH"):  # batch engines: warp (SMEM / L2), CTA (SMEM / L2), single-CTA
        n = int(rng.integers(1, 300)); b = int(rng.integers(1, 40))
        cb = rng.integers(0, hi, size=(b, n, n)).astype(np.int32)
        seed = int(rng.choice([KMB_SEED_BATCHED, KMB_SEED_KM]))
        refs = [O.ref_solve_batched_km(x) if seed == KMB_SEED_BATCHED else O.ref_solve_km(x) for x in cb]
        for eng in ([2, 3, 4, 6] if n <= 256 else []) + [8, 0]:
            s.set_option(OPT_ENGINE, eng)
            r = s.solve_batch(cb, seed)
            ok = all(np.array_equal(r.u[t], refs[t].u) and np.array_equal(r.v[t], refs[t].v)
                     and r.total_cost[t] == refs[t].total_cost for t in range(b))
            cases += 1
            if not ok:
                bad += 1
                print(f"MISMATCH batch b={b} n={n} hi={hi} seed={seed} engine={eng}", flush=True)
        continue
    n = int(rng.choice([rng.integers(1, 64), rng.integers(64, 300), rng.integers(300, 1500), rng.integers(1500, 3000)]))
    c = rng.integers(0, hi, size=(n, n)).astype(np.int32)
    seed = int(rng.choice([KMB_SEED_BATCHED, KMB_SEED_KM]))
    ref = O.ref_solve_batched_km(c) if seed == KMB_SEED_BATCHED else O.ref_solve_km(c)
    engines = [1, 5] + ([4, 6] if n <= 256 else []) + ([8] if n <= 4096 else [])
    for eng in engines:
        s.set_option(OPT_ENGINE, eng)
        r1 = s.solve(c, seed)
        r2 = s.solve(c, seed)
        ok = (np.array_equal(r1.u, ref.u) and np.array_equal(r1.v, ref.v) and r1.total_cost == ref.total_cost
              and np.array_equal(r1.row_to_col, r2.row_to_col) and r1.stats["rounds"] == r2.stats["rounds"])
        cases += 1
        if not ok:
            bad += 1
            print(f"MISMATCH n={n} hi={hi} seed={seed} engine={eng} duals={np.array_equal(r1.u, ref.u) and np.array_equal(r1.v, ref.v)} "
                  f"tot={r1.total_cost}/{ref.total_cost} det={np.array_equal(r1.row_to_col, r2.row_to_col)}", flush=True)
s.set_option(OPT_ENGINE, 0)
print(f"stress: {cases} engine runs, {bad} mismatches, {time.time()-t0:.0f} s", flush=True)
