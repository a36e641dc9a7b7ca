"""Replicated cluster engine (11): parity on random instances and configs 1, 2,
4 vs the reference / goldens, and timing by cluster size."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
from paper_2005_01182_b200 import Solver, workloads as W, KMB_SEED_BATCHED, KMB_SEED_KM
from paper_2005_01182_b200.api import OPT_ENGINE, OPT_MAX_CTAS
s = Solver(0)
s.set_option(OPT_ENGINE, 11)
rng = np.random.default_rng(1)
bad = 0
for t in range(int(os.environ.get("RAND", "60"))):
    n = int(rng.choice([rng.integers(1, 40), rng.integers(40, 600), rng.integers(600, 2000)]))
    hi = int(rng.choice([2, 100, 10**6]))
    c = rng.integers(0, hi, size=(n, n)).astype(np.int32)
    seed = int(rng.choice([KMB_SEED_BATCHED, KMB_SEED_KM]))
    G = int(rng.choice([1, 2, 4, 8, 16]))
    s.set_option(OPT_MAX_CTAS, G)
    ref = O.ref_solve_batched_km(c) if seed == 1 else O.ref_solve_km(c)
    r = s.solve(c, seed)
    ok = r.total_cost == ref.total_cost and np.array_equal(r.u, ref.u) and np.array_equal(r.v, ref.v)
    if not ok:
        bad += 1
        print("MISMATCH", n, hi, seed, G, r.total_cost, ref.total_cost, flush=True)
print("random:", bad, "mismatches", flush=True)
g = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "configs.json")))
for key in ("c1", "c2", "c4"):
    c = W.CONFIGS[key].make(); n = c.shape[0]
    dc = torch.from_numpy(c).cuda()
    r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
    for G in (4, 8, 16):
        s.set_option(OPT_MAX_CTAS, G)
        ts = [s.solve_into(dc, n, n, 1, r2c, u, v, tot) for _ in range(2)]
        ok = int(tot[0]) == g[key]["total_cost"] and W.fnv1a64(u.cpu().numpy()) == g[key]["u_fnv"] and W.fnv1a64(v.cpu().numpy()) == g[key]["v_fnv"]
        print(f"{key} G={G}: {min(x.seconds for x in ts)*1e3:.2f} ms rounds {ts[-1].rounds} ok={ok} engine={ts[-1].engine}", flush=True)
