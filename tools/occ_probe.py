"""Config 3 on the warp engine by resident warps per SM: stream-ordered call time
(L2 flushed) and per-instance durations (globaltimer), to size a dynamic
instance queue.  WPS=0,12,16,... (0 = auto); BATCHES=4096,2048."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE, OPT_WARPS_PER_SM
s = Solver(0)
st_ = torch.cuda.current_stream(); s.set_stream(st_.cuda_stream)
full = W.CONFIGS["c3"].make()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
s.set_option(OPT_ENGINE, int(os.environ.get("ENGINE", "4")))
ref = None
for b in [int(x) for x in os.environ.get("BATCHES", "4096,2048").split(",")]:
    c = torch.from_numpy(full[:b].copy()).cuda(); n = 128
    r2c = torch.empty((b, n), dtype=torch.int32, device="cuda"); u = torch.empty((b, n), dtype=torch.int64, device="cuda")
    v = torch.empty_like(u); tot = torch.empty(b, dtype=torch.int64, device="cuda")
    status = torch.zeros(b, dtype=torch.int32, device="cuda")
    for wps in [int(x) for x in os.environ.get("WPS", "0,12,16,20,24").split(",")]:
        s.set_option(OPT_WARPS_PER_SM, wps)
        for _ in range(3): s.solve_batch_into(c, b, n, 1, r2c, u, v, tot)
        ts = []
        for k in range(10):
            flush.fill_(k)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st_)
            s.solve_batch_async(c, b, n, 1, r2c, u, v, tot, status)
            e1.record(st_)
            torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        s.solve_batch_into(c, b, n, 1, r2c, u, v, tot)
        x = s.last_instance_stats(b)
        dur = (x[:, 10] - x[:, 9]) / 1e3
        t1 = (x[:, 10] - x[:, 9].min()) / 1e3
        if b == 4096:
            if ref is None: ref = tot.clone()
            ok = "" if torch.equal(tot, ref) else " MISMATCH"
        else:
            ok = ""
        print(f"batch {b} wps {wps}: {np.median(ts):.3f} ms (min {min(ts):.3f}){ok}; dur us p10 {np.percentile(dur,10):.0f} "
              f"p50 {np.median(dur):.0f} p90 {np.percentile(dur,90):.0f} max {dur.max():.0f} mean {dur.mean():.0f}; "
              f"end max {t1.max():.0f} us; rounds mean {x[:,3].mean():.0f}", flush=True)
s.set_option(OPT_WARPS_PER_SM, 0)
