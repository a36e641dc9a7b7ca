import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0); s.set_option(OPT_ENGINE, 8)
c = W.CONFIGS[os.environ.get("CFG", "c2")].make(); n = c.shape[0]
dc = torch.from_numpy(c).cuda()
r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
st = s.solve_into(dc, n, n, 1, r2c, u, v, tot)
print(f"{st.seconds*1e3:.2f} ms", int(tot[0]))
