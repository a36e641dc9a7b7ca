"""A/B CTA-engine builds (KMB_LIB per process): 512 / 1024 shards and c1."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import torch
    from paper_2005_01182_b200 import Solver, workloads as W
    from paper_2005_01182_b200.api import OPT_ENGINE
    s = Solver(0); s.set_option(OPT_ENGINE, 6)
    full = W.CONFIGS["c3"].make(); out = {"lib": os.path.basename(os.environ["KMB_LIB"])}
    for b in (512, 1024):
        c = torch.from_numpy(full[:b].copy()).cuda(); n = 128
        r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
        v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
        out[f"b{b}"] = round(min(s.solve_batch_into(c, b, n, 1, r2c, u, v, tot).seconds for _ in range(8)) * 1e3, 3)
    c1 = W.CONFIGS["c1"].make(); n = 256
    d = torch.from_numpy(c1).cuda(); r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
    out["c1"] = round(min(s.solve_into(d, n, n, 1, r2c, u, v, tot).seconds for _ in range(8)) * 1e3, 3)
    print(json.dumps(out))
else:
    for lib in sys.argv[1:]:
        env = dict(os.environ, KMB_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-1500:], flush=True)
