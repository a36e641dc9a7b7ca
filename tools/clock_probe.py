"""SM clock under the config-3 kernel: loop solves ~3 s while sampling nvidia-smi."""
import os, sys, subprocess, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
s = Solver(0)
c = W.CONFIGS["c3"].make(); b, n, _ = c.shape
dc = torch.from_numpy(c).cuda()
r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
t0 = time.time(); k = 0; ts = []
while time.time() - t0 < 3.0:
    st = s.solve_batch_into(dc, b, n, 1, r2c, u, v, tot); ts.append(st.seconds); k += 1
p.terminate(); out = p.communicate()[0].strip().splitlines()
clk = [float(l.split(",")[0]) for l in out if l.strip()]
print(f"solves={k} median kernel {statistics.median(ts)*1e3:.3f} ms; sm clock median {statistics.median(clk):.0f} MHz min {min(clk):.0f} max {max(clk):.0f}; samples={len(clk)}; last={out[-3:]}")
