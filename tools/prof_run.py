"""Small profiling driver: warm-up + 2 solves of one config (for ncu)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--batch", type=int, default=4096)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--engine", type=int, default=0)
ap.add_argument("--maxg", type=int, default=0)
a = ap.parse_args()
s = Solver(0)
s.set_option(OPT_ENGINE, a.engine)
from paper_2005_01182_b200.api import OPT_MAX_CTAS
s.set_option(OPT_MAX_CTAS, a.maxg)
if os.environ.get("RES16"): s.set_option(7, int(os.environ["RES16"]))
c = W.CONFIGS[a.config].make(batch=a.batch) if a.config == "c3" else W.CONFIGS[a.config].make()
dc = torch.from_numpy(c).cuda()
if a.config == "c3":
    b, n, _ = c.shape
    r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
    for _ in range(a.iters):
        st = s.solve_batch_into(dc, b, n, 1, r2c, u, v, tot)
else:
    n = c.shape[0]
    r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
    for _ in range(a.iters):
        st = s.solve_into(dc, n, n, 1, r2c, u, v, tot)
from paper_2005_01182_b200.api import _stats_dict
d = _stats_dict(st); print(a.config, d, "us/round", {k: round(x / 1e3 / max(d["rounds"], 1), 2) for k, x in zip(["relax", "b1", "absorb", "b2", "end", "b3"], d["stage_ns"])})
