"""A/B single-instance configs (c2, c4, c5) across libkmb.so variants (KMB_LIB per process)."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import torch
    from paper_2005_01182_b200 import Solver, workloads as W
    s = Solver(0)
    out = {"lib": os.path.basename(os.environ.get("KMB_LIB", "default"))}
    for key in os.environ.get("CFGS", "c5,c4,c2").split(","):
        c = W.CONFIGS[key].make(); n = c.shape[0]
        dc = torch.from_numpy(c).cuda()
        r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
        v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
        ts = [s.solve_into(dc, n, n, 1, r2c, u, v, tot).seconds for _ in range(int(os.environ.get("REPS", "3")))]
        out[key] = round(min(ts) * 1e3, 2); out[key + "_tot"] = int(tot[0])
        del dc
    print(json.dumps(out))
else:
    for lib in sys.argv[1:]:
        env = dict(os.environ, KMB_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-1500:], flush=True)
