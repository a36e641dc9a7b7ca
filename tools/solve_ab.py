"""A/B grid/cluster engine builds (KMB_LIB per process): c4 (cluster) and c5 (grid)."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    from paper_2005_01182_b200 import Solver, workloads as W
    s = Solver(0)
    out = {"lib": os.path.basename(os.environ["KMB_LIB"])}
    for key in os.environ.get("CFGS", "c4,c5").split(","):
        c = W.CONFIGS[key].make(); n = c.shape[0]; d = torch.from_numpy(c).cuda()
        r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
        v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
        out[key] = round(min(s.solve_into(d, n, n, 1, r2c, u, v, tot).seconds for _ in range(2)) * 1e3, 2)
        out[key + "_tot"] = int(tot[0])
        del d
        torch.cuda.empty_cache()
    print(json.dumps(out))
else:
    for lib in sys.argv[1:]:
        env = dict(os.environ, KMB_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-1500:], flush=True)
