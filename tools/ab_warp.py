"""A/B the warp engine's residency bound on config 3."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE, OPT_WARPS_PER_SM
s = Solver(0)
c = W.CONFIGS["c3"].make()
b, n, _ = c.shape
dc = torch.from_numpy(c).cuda()
r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
ref = None
for eng in [int(x) for x in os.environ.get("ENGINES", "4").split(",")]:
  for wps in [int(x) for x in os.environ.get("WPS", "0,4,8,12,16,24").split(",")]:
    s.set_option(OPT_ENGINE, eng); s.set_option(OPT_WARPS_PER_SM, wps)
    ts = []
    for it in range(6):
        flush.fill_(it)
        st = s.solve_batch_into(dc, b, n, 1, r2c, u, v, tot)
        ts.append(st.seconds)
    if ref is None: ref = tot.clone()
    print(f"engine {eng} warps/SM {wps:2d}: {min(ts)*1e3:.3f} ms ({b/min(ts)/1e6:.2f}M solves/s) same={bool(torch.equal(tot, ref))} inst_cycles mean={st.sum_instance_cycles/b/1e3:.0f}k max={st.max_instance_cycles/1e3:.0f}k stages/inst(k)={[round(x/b/1e3) for x in st.stage_ns[:4]]} rounds/inst={st.rounds/b:.0f} rows/inst={st.rows_scanned/b:.0f}", flush=True)
from paper_2005_01182_b200.api import OPT_U16
for uu in (0, 1):
    s.set_option(OPT_ENGINE, 4); s.set_option(OPT_WARPS_PER_SM, 0); s.set_option(OPT_U16, uu)
    ts = []
    for it in range(6):
        flush.fill_(it)
        st = s.solve_batch_into(dc, b, n, 1, r2c, u, v, tot)
        ts.append(st.seconds)
    print(f"engine 4 u16={uu}: {min(ts)*1e3:.3f} ms ({b/min(ts)/1e6:.2f}M solves/s) same={bool(torch.equal(tot, ref))} inst_cycles mean={st.sum_instance_cycles/b/1e3:.0f}k max={st.max_instance_cycles/1e3:.0f}k stages/inst(k)={[round(x/b/1e3) for x in st.stage_ns[:4]]}", flush=True)
