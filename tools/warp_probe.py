"""Per-round stage cycles of the warp engine by batch size (build with -DKMB_WARP_STAGE_CLOCKS=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
full = W.CONFIGS["c3"].make()
for eng in [int(x) for x in os.environ.get("ENGS", "4,3").split(",")]:
    for b in [int(x) for x in os.environ.get("BATCHES", "512,1024,2048,4096").split(",")]:
        first = int(os.environ.get("FIRST", "0")) if b == 1 else 0
        c = torch.from_numpy(full[first:first + b].copy()).cuda(); n = 128
        r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
        v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
        s.set_option(OPT_ENGINE, eng)
        for _ in range(3): st = s.solve_batch_into(c, b, n, 1, r2c, u, v, tot)
        x = s.last_instance_stats(b)
        R = x[:, 3].sum()
        print(f"e{eng} batch {b}: {st.seconds*1e3:.3f} ms, cycles/round: relax {x[:,5].sum()/R:.0f} min {x[:,6].sum()/R:.0f} absorb {x[:,7].sum()/R:.0f} epoch {x[:,8].sum()/R:.0f}; inst cycles mean {x[:,4].mean()/1e3:.0f}k max {x[:,4].max()/1e3:.0f}k; rounds mean {x[:,3].mean():.0f} max {x[:,3].max()}; ns/round of the longest {(x[:,10]-x[:,9])[x[:,3].argmax()]/x[:,3].max():.0f}", flush=True)
