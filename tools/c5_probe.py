"""Config 5 (and 4) on the grid / cluster engines and the device-exchange
sharded engine (ranks as CTA groups on this GPU): best-of-3 device times,
golden checks."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W

g = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "configs.json")))
s = Solver(0)
out = {}
for key in os.environ.get("CFGS", "c5,c4").split(","):
    c = W.CONFIGS[key].make(); n = c.shape[0]
    dc = torch.from_numpy(c).cuda()
    r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
    sts = [s.solve_into(dc, n, n, 1, r2c, u, v, tot) for _ in range(3)]
    ok = int(tot[0]) == g[key]["total_cost"] and W.fnv1a64(u.cpu().numpy()) == g[key]["u_fnv"]
    out[key] = {"ms": round(min(x.seconds for x in sts) * 1e3, 2), "ok": ok, "engine": sts[0].engine,
                "us_per_round": {k: round(x / 1e3 / sts[-1].rounds, 2) for k, x in
                                 zip(["relax", "b1", "absorb", "b2", "end", "b3"], sts[-1].stage_ns)}}
    if key == "c5":
        for R in (1, 2, 4):
            rs = [s.solve_sharded_local(dc, R) for _ in range(2)]
            out[f"{key}_sharded_{R}"] = {"ms": round(min(x.stats["seconds"] for x in rs) * 1e3, 2),
                                         "ok": rs[-1].total_cost == g[key]["total_cost"] and W.fnv1a64(rs[-1].u) == g[key]["u_fnv"]}
    del dc
    torch.cuda.empty_cache()
print(json.dumps(out))
