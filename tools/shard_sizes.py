"""Config-3 shard sizes (4096/N instances per GPU for N = 1, 2, 4, 8): device
time per engine, to pick the engine per shard size."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE, OPT_WARPS_PER_SM
s = Solver(0)
full = W.CONFIGS["c3"].make()
for b in (4096, 2048, 1024, 512):
    c = torch.from_numpy(full[:b].copy()).cuda()
    n = 128
    r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
    res = {"batch": b}
    ref = None
    for eng in (4, 3, 6, 2):
        s.set_option(OPT_ENGINE, eng)
        ts = [s.solve_batch_into(c, b, n, 1, r2c, u, v, tot).seconds for _ in range(5)]
        res[f"e{eng}_ms"] = round(min(ts) * 1e3, 3)
        if ref is None: ref = tot.clone()
        res[f"e{eng}_ok"] = bool(torch.equal(tot, ref))
    print(json.dumps(res), flush=True)
