"""A/B single-CTA engine builds (KMB_LIB per process): c2 and c4 on engine 8, and
a batch of 64 n = 512 instances."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    from paper_2005_01182_b200 import Solver, workloads as W
    from paper_2005_01182_b200.api import OPT_ENGINE
    s = Solver(0); s.set_option(OPT_ENGINE, 8)
    out = {"lib": os.path.basename(os.environ["KMB_LIB"])}
    for key in ("c2", "c4"):
        c = W.CONFIGS[key].make(); n = c.shape[0]; d = torch.from_numpy(c).cuda()
        r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
        v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
        out[key] = round(min(s.solve_into(d, n, n, 1, r2c, u, v, tot).seconds for _ in range(3)) * 1e3, 2)
    b, n = 64, 512
    c = np.random.default_rng(5).integers(0, 10**6, (b, n, n)).astype(np.int32); d = torch.from_numpy(c).cuda()
    r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
    out["b64n512"] = round(min(s.solve_batch_into(d, b, n, 1, r2c, u, v, tot).seconds for _ in range(3)) * 1e3, 2)
    out["tot"] = int(tot.sum())
    print(json.dumps(out))
else:
    for lib in sys.argv[1:]:
        env = dict(os.environ, KMB_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-1500:], flush=True)
