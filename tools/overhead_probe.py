"""Host overhead of one kmb_solve_batch_i32 call: outer CUDA events (what
bench.py times) vs the library's own kernel events (stats.seconds)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
s = Solver(0)
st_ = torch.cuda.current_stream(); s.set_stream(st_.cuda_stream)
full = W.CONFIGS["c3"].make()
for b in (4096, 512):
    c = torch.from_numpy(full[:b].copy()).cuda(); n = 128
    r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
    for _ in range(3): s.solve_batch_into(c, b, n, 1, r2c, u, v, tot)
    outer, inner, wall = [], [], []
    for k in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(st_); st = s.solve_batch_into(c, b, n, 1, r2c, u, v, tot); e1.record(st_)
        torch.cuda.synchronize()
        wall.append((time.perf_counter() - t0) * 1e3)
        outer.append(e0.elapsed_time(e1)); inner.append(st.seconds * 1e3)
    f = lambda x: sum(x) / len(x)
    print(f"batch {b}: outer {f(outer):.3f} ms, kernel {f(inner):.3f} ms, overhead {f(outer)-f(inner):.3f} ms, host wall {f(wall):.3f} ms", flush=True)
