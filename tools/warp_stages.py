"""Config-3 batch on the warp engine: device time and, with a stage-clock build
(-DKMB_WARP_STAGE_CLOCKS=1), SM cycles per stage summed over instances
(relax of ordinary rounds, min + absorb, epoch-start re-relax, epoch end).
Env: KMB_LIB, U16=0/1, BATCH."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE, OPT_U16
s = Solver(0)
s.set_option(OPT_ENGINE, 4)
s.set_option(OPT_U16, int(os.environ.get("U16", "0")))
b = int(os.environ.get("BATCH", "4096"))
c = W.CONFIGS["c3"].make(batch=b)
n = c.shape[1]
dc = torch.from_numpy(c).cuda()
r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
ts = []
for k in range(8):
    st = s.solve_batch_into(dc, b, n, 1, r2c, u, v, tot)
    ts.append(st.seconds)
ist = s.last_instance_stats(b)
ts = sorted(ts[2:])
cyc = ist[:, 4].astype(np.float64)
out = {"lib": os.environ.get("KMB_LIB", "default"), "u16": os.environ.get("U16", "0"),
       "median_ms": 1e3 * ts[len(ts) // 2], "epochs": float(ist[:, 0].mean()), "dual_steps": float(ist[:, 1].mean()),
       "rows": float(ist[:, 2].mean()), "rounds": float(ist[:, 3].mean()), "rounds_max": int(ist[:, 3].max()),
       "cycles_mean": float(cyc.mean()), "cycles_max": float(cyc.max()),
       "stage_frac": {k: float(ist[:, 5 + i].sum() / cyc.sum()) for i, k in enumerate(["relax", "min_absorb", "estart_relax", "epoch_end"])},
       "hash": W.fnv1a64(np.concatenate([tot.cpu().numpy(), u.cpu().numpy().ravel()]))}
print(json.dumps(out), flush=True)
