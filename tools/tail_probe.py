"""Config-3 warp engine tail: when instances finish, and whether the slowest
ones are long chains (rounds) or slow rounds."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
c = W.CONFIGS["c3"].make(); b, n, _ = c.shape
dc = torch.from_numpy(c).cuda()
r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
for eng in [int(e) for e in os.environ.get("ENGINES", "4,6").split(",")]:
    s.set_option(OPT_ENGINE, eng)
    for _ in range(3): st = s.solve_batch_into(dc, b, n, 1, r2c, u, v, tot)
    x = s.last_instance_stats(b)
    t0 = x[:, 9] - x[:, 9].min(); t1 = x[:, 10] - x[:, 9].min(); dur = x[:, 10] - x[:, 9]
    rounds = x[:, 3]; rows = x[:, 2]
    print(f"engine {eng}: kernel {st.seconds*1e3:.3f} ms, span {t1.max()/1e3:.0f} us")
    print("  finish-time percentiles (us):", {p: round(np.percentile(t1, p) / 1e3) for p in (10, 50, 90, 99, 99.9, 100)})
    print("  rounds percentiles:", {p: int(np.percentile(rounds, p)) for p in (10, 50, 90, 99, 99.9, 100)})
    print("  rows percentiles:", {p: int(np.percentile(rows, p)) for p in (10, 50, 90, 99, 100)})
    print(f"  corr(dur, rounds) = {np.corrcoef(dur, rounds)[0,1]:.3f}, corr(dur, rows) = {np.corrcoef(dur, rows)[0,1]:.3f}")
    o = np.argsort(-dur)[:8]
    for i in o:
        print(f"   inst {i}: dur {dur[i]/1e3:.0f} us start {t0[i]/1e3:.0f} rounds {rounds[i]} rows {rows[i]} ns/round {dur[i]/rounds[i]:.0f}")
    m = rounds > 0
    print(f"  ns/round: median {np.median(dur[m]/rounds[m]):.0f}, for the 1% longest chains {np.median((dur/np.maximum(rounds,1))[rounds >= np.percentile(rounds, 99)]):.0f}")
