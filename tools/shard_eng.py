"""Config-3 shards: per-call time (L2 flushed) for chosen engines (ENGS)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE
s = Solver(0)
st_ = torch.cuda.current_stream(); s.set_stream(st_.cuda_stream)
full = W.CONFIGS["c3"].make()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
for b in [int(x) for x in os.environ.get("BATCHES", "4096,2048,1024,512").split(",")]:
    c = torch.from_numpy(full[:b].copy()).cuda(); n = 128
    r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
    status = torch.zeros(b, dtype=torch.int32, device="cuda")
    line = [f"batch {b}:"]
    ref = None
    for eng in [int(x) for x in os.environ.get("ENGS", "0,2,4,6").split(",")]:
        s.set_option(OPT_ENGINE, eng)
        for _ in range(3): st = s.solve_batch_into(c, b, n, 1, r2c, u, v, tot)
        ts = []
        for k in range(8):
            flush.fill_(k)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st_)
            if os.environ.get("ASYNC"):
                s.solve_batch_async(c, b, n, 1, r2c, u, v, tot, status)
            else:
                st = s.solve_batch_into(c, b, n, 1, r2c, u, v, tot)
            e1.record(st_)
            torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        if ref is None: ref = tot.clone()
        line.append(f"e{eng}->{st.engine} {sum(ts)/len(ts):.3f} ms{'' if torch.equal(tot, ref) else ' MISMATCH'}"
                    f"{' status!' if int(status.abs().sum()) else ''}")
    print("  ".join(line), flush=True)
s.set_option(OPT_ENGINE, 0)
