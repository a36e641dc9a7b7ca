"""Randomised stress: engines x sizes x value ranges x seeds against the
reference (duals, total cost) and against themselves (determinism: the same
matching and round count twice).  Usage: python tools/stress.py [seconds]
(BATCH=1: random batches through every batch engine instead; RES16=1: the warp
engine relaxing from its 16-bit resident copy, value ranges around the 16-bit
and narrow-key limits, rows and instances that do not fit; WIDE=1: int64
costs up to validate_instance's headroom through kmb_solve_i64 / the wide
engine; SHARD=1: the device-exchange column-sharded engine with 1-8 ranks as
CTA groups, against the reference and the grid engine's matching)."""
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
    if os.environ.get("RES16"):
        n = int(rng.integers(65, 257)); b = int(rng.integers(1, 24))
        h16 = int(rng.choice([100, 30000, 65534, 65535, 65536, 65537, 70000, 10**6, 2**21 - 1, 2**21, 2**23]))
        cb = rng.integers(0, h16 + 1, size=(b, n, n)).astype(np.int32)
        if rng.random() < 0.5:  # a few rows (sometimes many) leave the 16-bit range
            for t in range(b):
                k = int(rng.choice([0, 1, 2, n // 16, n // 16 + 3, n // 4]))
                if k:
                    rr = rng.choice(n, size=k, replace=False)
                    cb[t][rr, int(rng.integers(0, n))] += int(rng.choice([65535, 10**5, 10**6]))
        if rng.random() < 0.3:
            cb += int(rng.integers(0, 10**6))  # a common offset: the copy is relative to the row minimum
        seed = int(rng.choice([KMB_SEED_BATCHED, KMB_SEED_KM]))
        refs = [O.ref_solve_batched_km(x) if seed == KMB_SEED_BATCHED else O.ref_solve_km(x) for x in cb]
        s.set_option(OPT_ENGINE, 4)
        out = {}
        for mode in (1, -1):
            s.set_option(7, mode)
            out[mode] = r = s.solve_batch(cb, seed)
            ok = all(np.array_equal(r.u[t], refs[t].u) and np.array_equal(r.v[t], refs[t].v)
                     and r.total_cost[t] == refs[t].total_cost for t in range(b))
            cases += 1
            if not ok:
                bad += 1
                print(f"MISMATCH res16={mode} b={b} n={n} hi={h16} seed={seed}", flush=True)
        if not np.array_equal(out[1].row_to_col, out[-1].row_to_col):
            bad += 1
            print(f"MATCHING DIFFERS between modes b={b} n={n} hi={h16} seed={seed}", flush=True)
        continue
    if os.environ.get("BATCH"):  # batch engines: warp (SMEM / L2), CTA (SMEM / L2), single-CTA
        n = int(rng.integers(1, 300)); b = int(rng.integers(1, 40))
        cb = rng.integers(0, hi, size=(b, n, n)).astype(np.int32)
        seed = int(rng.choice([KMB_SEED_BATCHED, KMB_SEED_KM]))
        refs = [O.ref_solve_batched_km(x) if seed == KMB_SEED_BATCHED else O.ref_solve_km(x) for x in cb]
        for eng in ([4, 6] if n <= 256 else []) + [8, 0]:
            s.set_option(OPT_ENGINE, eng)
            r = s.solve_batch(cb, seed)
            ok = all(np.array_equal(r.u[t], refs[t].u) and np.array_equal(r.v[t], refs[t].v)
                     and r.total_cost[t] == refs[t].total_cost for t in range(b))
            cases += 1
            if not ok:
                bad += 1
                print(f"MISMATCH batch b={b} n={n} hi={hi} seed={seed} engine={eng}", flush=True)
        continue
    if os.environ.get("WIDE"):
        n = int(rng.integers(1, 400))
        head = ((1 << 62) // n) // (2 * n + 2)
        hw = int(rng.choice([2**29, 2**35, head]))
        c = rng.integers(0, min(hw, head), size=(n, n), dtype=np.int64)
        c[rng.random((n, n)) < 0.3] = int(rng.integers(0, 100))
        seed = int(rng.choice([KMB_SEED_BATCHED, KMB_SEED_KM]))
        mx = max(int(c.max()), 1)
        ref = (O.ref_solve_km(c) if seed == KMB_SEED_KM else
               O.ref_solve_batched_km(c) if mx * mx < 2**63 else O.kmo_solve_batched(c))
        r = s.solve(c, seed)
        cases += 1
        if not (np.array_equal(r.u, ref.u) and np.array_equal(r.v, ref.v) and r.total_cost == ref.total_cost):
            bad += 1
            print(f"MISMATCH wide n={n} max={mx} seed={seed} engine={r.stats['engine']}", flush=True)
        continue
    if os.environ.get("SHARD"):
        n = int(rng.choice([rng.integers(1, 64), rng.integers(64, 700), rng.integers(700, 3000)]))
        c = rng.integers(0, hi, size=(n, n)).astype(np.int32)
        seed = int(rng.choice([KMB_SEED_BATCHED, KMB_SEED_KM]))
        ref = O.ref_solve_batched_km(c) if seed == KMB_SEED_BATCHED else O.ref_solve_km(c)
        s.set_option(OPT_ENGINE, 1)
        g = s.solve(c, seed)
        for R in (1, 2, 3, 5, 8):
            r = s.solve_sharded_local(c, R, seed)
            cases += 1
            if not (np.array_equal(r.u, ref.u) and np.array_equal(r.v, ref.v) and r.total_cost == ref.total_cost
                    and np.array_equal(r.row_to_col, g.row_to_col)):
                bad += 1
                print(f"MISMATCH sharded n={n} hi={hi} seed={seed} ranks={R}", flush=True)
        continue
    n = int(rng.choice([rng.integers(1, 64), rng.integers(64, 300), rng.integers(300, 1500), rng.integers(1500, 3000)]))
    c = rng.integers(0, hi, size=(n, n)).astype(np.int32)
    seed = int(rng.choice([KMB_SEED_BATCHED, KMB_SEED_KM]))
    ref = O.ref_solve_batched_km(c) if seed == KMB_SEED_BATCHED else O.ref_solve_km(c)
    engines = [1, 5] + ([4, 6] if n <= 256 else []) + ([8] if n <= 4096 else []) + ([11] if n <= 5120 else [])
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
