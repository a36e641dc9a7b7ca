"""Config 4 (n = 4096) by engine and CTA count (KMB_OPT_MAX_CTAS)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE, OPT_MAX_CTAS
s = Solver(0)
c = W.CONFIGS[os.environ.get("CFG", "c4")].make(); n = c.shape[0]
dc = torch.from_numpy(c).cuda()
r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
ref = None
for spec in os.environ.get("SPECS", "5:4,5:8,5:16,1:16,1:32,1:64,1:128,8:0").split(","):
    eng, g = (int(x) for x in spec.split(":"))
    s.set_option(OPT_ENGINE, eng); s.set_option(OPT_MAX_CTAS, g)
    ts = [s.solve_into(dc, n, n, 1, r2c, u, v, tot) for _ in range(2)]
    t = min(x.seconds for x in ts)
    if ref is None: ref = int(tot[0])
    print(f"engine {eng} max_ctas {g}: {t*1e3:.1f} ms, rounds {ts[-1].rounds}, us/round {t*1e6/max(ts[-1].rounds,1):.2f}, same={int(tot[0]) == ref}", flush=True)
