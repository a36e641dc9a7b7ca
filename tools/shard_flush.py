"""Config-3 shard sizes with an L2 flush before every solve (as bench.py times them)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
s = Solver(0)
st_ = torch.cuda.current_stream(); s.set_stream(st_.cuda_stream)
full = W.CONFIGS["c3"].make()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
for b in (4096, 2048, 1024, 512):
    c = torch.from_numpy(full[:b].copy()).cuda(); n = 128
    r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
    for _ in range(3): s.solve_batch_into(c, b, n, 1, r2c, u, v, tot)
    ts = []; tn = []
    for k in range(10):
        flush.fill_(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st_); st = s.solve_batch_into(c, b, n, 1, r2c, u, v, tot); e1.record(st_)
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        e0.record(st_); s.solve_batch_into(c, b, n, 1, r2c, u, v, tot); e1.record(st_)
        torch.cuda.synchronize(); tn.append(e0.elapsed_time(e1))
    print(f"batch {b}: engine {st.engine} flushed {sum(ts)/len(ts):.3f} ms, warm {sum(tn)/len(tn):.3f} ms -> job rate at {4096//b} GPUs {4096/(sum(ts)/len(ts))/1e3:.2f} M/s", flush=True)
