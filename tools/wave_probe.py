"""Per-instance start/end times of the config-3 batch engines (globaltimer)."""
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
for eng, u16 in [(int(e.split(':')[0]), int(e.split(':')[1])) for e in os.environ.get('ENGINES', '4:0').split(',')]:
    s.set_option(OPT_ENGINE, eng); s.set_option(5, u16)
    for _ in range(3): st = s.solve_batch_into(dc, b, n, 1, r2c, u, v, tot)
    x = s.last_instance_stats(b)
    t0 = x[:, 9] - x[:, 9].min(); t1 = x[:, 10] - x[:, 9].min(); dur = x[:, 10] - x[:, 9]
    print(f"engine {eng} u16 {u16}: kernel {st.seconds*1e3:.3f} ms; span {t1.max()/1e6:.3f} ms; start p50 {np.median(t0)/1e3:.1f} us p99 {np.percentile(t0,99)/1e3:.1f} us max {t0.max()/1e3:.1f} us; dur p50 {np.median(dur)/1e3:.1f} us p99 {np.percentile(dur,99)/1e3:.1f} max {dur.max()/1e3:.1f} us; cycles max {x[:,4].max()/1e3:.0f}k => {x[:,4].max()/1.965e3:.1f} us at 1965MHz")
    late = (t0 > 100e3).sum(); print("instances starting >100us late:", late)
    names = ["epochs", "dual_steps", "rows", "rounds", "cycles", "c_relax", "c_min", "c_absorb", "c_epoch"]
    print("  ".join(f"{k}={x[:, i].mean():.1f}" for i, k in enumerate(names)))
    print("per round: " + "  ".join(f"{k}={x[:, i].sum() / x[:, 3].sum():.1f}" for i, k in enumerate(names) if i != 3))
