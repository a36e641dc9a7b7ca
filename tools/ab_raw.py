"""A/B of library builds through raw ctypes (libraries whose ABI predates the
current Python binding): configs solved on the auto engine, best of REPS,
each library in its own process.  Usage: CFGS=c4,c5 python tools/ab_raw.py lib1.so lib2.so ..."""
import ctypes as C, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 2 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import torch
    from paper_2005_01182_b200 import workloads as W
    from paper_2005_01182_b200.api import Stats
    lib = C.CDLL(sys.argv[2])
    h = C.c_void_p()
    assert lib.kmb_create(0, C.byref(h)) == 0
    lib.kmb_set_option(h, 3, C.c_int64(int(os.environ.get("ENGINE", "0"))))
    out = {"lib": os.path.basename(sys.argv[2])}
    for key in os.environ.get("CFGS", "c4,c5").split(","):
        if key.startswith("u"):  # uN: uniform U{0..1e6} instance of size N
            import numpy as np
            n = int(key[1:]); c = np.random.default_rng(n).integers(0, 10**6, (n, n)).astype(np.int32)
        else:
            c = W.CONFIGS[key].make(); n = c.shape[0]
        d = torch.from_numpy(c).cuda()
        r2c = torch.empty(n, dtype=torch.int32, device="cuda"); u = torch.empty(n, dtype=torch.int64, device="cuda")
        v = torch.empty_like(u); tot = torch.empty(1, dtype=torch.int64, device="cuda")
        ts = []
        for _ in range(int(os.environ.get("REPS", "3"))):
            st = Stats()
            rc = lib.kmb_solve_i32(h, C.c_void_p(d.data_ptr()), n, C.c_int64(n), 1, C.c_double(0.0),
                                   C.c_void_p(r2c.data_ptr()), C.c_void_p(u.data_ptr()), C.c_void_p(v.data_ptr()),
                                   C.c_void_p(tot.data_ptr()), C.byref(st))
            assert rc == 0
            ts.append(st.seconds)
        out[key] = round(min(ts) * 1e3, 2); out[key + "_tot"] = int(tot[0])
        del d
        torch.cuda.empty_cache()
    print(json.dumps(out))
else:
    for lib in sys.argv[1:]:
        r = subprocess.run([sys.executable, __file__, "--child", os.path.abspath(lib)], capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-1500:], flush=True)
