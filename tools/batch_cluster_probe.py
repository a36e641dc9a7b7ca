import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle as O
from paper_2005_01182_b200 import Solver
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
for b, n in ((4, 3072), (9, 2500), (12, 2500)):
    c = np.random.default_rng(b).integers(0, 10**6, (b, n, n)).astype(np.int32)
    d = torch.from_numpy(c).cuda()
    o = [torch.empty((b, n), dtype=torch.int32, device="cuda"), torch.empty((b, n), dtype=torch.int64, device="cuda"),
         torch.empty((b, n), dtype=torch.int64, device="cuda"), torch.empty(b, dtype=torch.int64, device="cuda")]
    for eng in (8, 0):
        s.set_option(OPT_ENGINE, eng)
        st = min((s.solve_batch_into(d, b, n, 1, *o) for _ in range(2)), key=lambda x: x.seconds)
        print(b, n, "engine", eng, "->", st.engine, round(st.seconds * 1e3, 2), "ms", flush=True)
    ref = O.ref_solve_batched_km(c[0])
    assert int(o[3][0]) == ref.total_cost and np.array_equal(o[1][0].cpu().numpy(), ref.u)
print("ok")
