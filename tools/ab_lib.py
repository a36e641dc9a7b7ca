"""A/B the config-3 batch solve across libkmb.so variants: each variant runs in
its own process (KMB_LIB), median device time over REPS solves."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    from paper_2005_01182_b200 import Solver, workloads as W
    from paper_2005_01182_b200.api import OPT_ENGINE
    key = os.environ.get("CFG", "c3"); eng = int(os.environ.get("ENGINE", "0"))
    s = Solver(0)
    if eng: s.set_option(OPT_ENGINE, eng)
    if os.environ.get("RES16"): s.set_option(7, int(os.environ["RES16"]))
    if key.startswith("u"):  # uNxB[xH]: B uniform U{0..H} (100000) instances of size N
        nn, bb, *hi = map(int, key[1:].split("x"))
        c = np.random.default_rng(1).integers(0, (hi[0] if hi else 100000) + 1, size=(bb, nn, nn), dtype=np.int32)
    else:
        c = W.CONFIGS[key].make(batch=int(os.environ["MAKE_BATCH"])) if os.environ.get("MAKE_BATCH") else W.CONFIGS[key].make()
    if c.ndim == 2: c = c[None]
    if os.environ.get("BATCH"): c = np.ascontiguousarray(c[:int(os.environ["BATCH"])])
    b, n, _ = c.shape
    dc = torch.from_numpy(c).cuda()
    r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
    ts = []
    for k in range(int(os.environ.get("REPS", "15"))):
        st = (s.solve_batch_into(dc, b, n, 1, r2c, u, v, tot) if b > 1 else s.solve_into(dc, n, n, 1, r2c, u, v, tot))
        ts.append(st.seconds)
    ts = sorted(ts[2:])
    print(json.dumps({"lib": os.environ.get("KMB_LIB", "default"), "cfg": key, "median_ms": ts[len(ts) // 2] * 1e3, "min_ms": ts[0] * 1e3, "tot0": int(tot[0]),
                      "hash": W.fnv1a64(np.concatenate([tot.cpu().numpy(), u.cpu().numpy().ravel(), r2c.cpu().numpy().ravel().astype(np.int64)]))}))
else:
    for lib in sys.argv[1:]:
        env = dict(os.environ, KMB_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(out.stdout.strip() or out.stderr[-2000:], flush=True)
