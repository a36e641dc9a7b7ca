"""Full-frontier scan microbenchmark + one solve per config (grid engine)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE, _stats_dict
s = Solver(0)
engines = [int(x) for x in os.environ.get("ENGINES", "1").split(",")]
for key in sys.argv[1:] or ["c5"]:
    c = W.CONFIGS[key].make()
    n = c.shape[0]
    dc = torch.from_numpy(c).cuda()
    t, g = s.bench_scan(dc, n, n, 5)
    for eng in engines:
      s.set_option(OPT_ENGINE, eng)
      r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
      v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
      for _ in range(2):
        st = s.solve_into(dc, n, n, 1, r2c, u, v, tot)
      d = _stats_dict(st)
      alg = 4.0 * n * (d["rows_scanned"] + 2 * n)
      print(f"{key} e{eng}: scan pass {t*1e3:.3f} ms = {g:.0f} GB/s | solve {d['seconds']*1e3:.1f} ms rounds={d['rounds']} phases={d['phases']} ds={d['dual_steps']} eff={alg/d['seconds']/1e9:.0f} GB/s relax-stage={4.0*n*d['rows_scanned']/(d['stage_ns'][0]*1e-9)/1e9:.0f} GB/s us/round={[round(x/1e3/d['rounds'],2) for x in d['stage_ns']]}", flush=True)
