"""Per-round stage cycles of the CTA engine (build with -DKMB_CTA_STAGE_CLOCKS=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
full = W.CONFIGS["c3"].make()
for b in [int(x) for x in os.environ.get("BATCHES", "512,1024,4096").split(",")]:
    c = torch.from_numpy(full[:b].copy()).cuda(); n = 128
    r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
    for eng in (6,):
        s.set_option(OPT_ENGINE, eng)
        for _ in range(3): st = s.solve_batch_into(c, b, n, 1, r2c, u, v, tot)
        x = s.last_instance_stats(b)
        R = x[:, 3].sum()
        print(f"batch {b} e{eng}: {st.seconds*1e3:.3f} ms, rounds/inst {R/b:.0f}, cycles/round: relax {x[:,5].sum()/R:.0f} min {x[:,6].sum()/R:.0f} absorb {x[:,7].sum()/R:.0f} epoch {x[:,8].sum()/R:.0f}; max inst cycles {x[:,4].max()/1e3:.0f}k", flush=True)
