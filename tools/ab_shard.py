"""A/B a config-3 shard size across libkmb.so variants (KMB_LIB per process)."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import torch
    from paper_2005_01182_b200 import Solver, workloads as W
    from paper_2005_01182_b200.api import OPT_ENGINE
    s = Solver(0)
    full = W.CONFIGS["c3"].make()
    out = {"lib": os.path.basename(os.environ.get("KMB_LIB", "default"))}
    for b in [int(x) for x in os.environ.get("BATCHES", "512,1024").split(",")]:
        c = torch.from_numpy(full[:b].copy()).cuda(); n = 128
        r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
        v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
        for eng in [int(x) for x in os.environ.get("ENGS", "6").split(",")]:
            s.set_option(OPT_ENGINE, eng)
            ts = [s.solve_batch_into(c, b, n, 1, r2c, u, v, tot).seconds for _ in range(7)]
            out[f"b{b}_e{eng}"] = round(min(ts) * 1e3, 3)
    print(json.dumps(out))
else:
    for lib in sys.argv[1:]:
        env = dict(os.environ, KMB_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-1500:], flush=True)
