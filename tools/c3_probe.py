"""Config-3 probes on one GPU: device time of the stream-ordered call with the
options given, and the end-to-end time through the synchronous call with
pinned and with pageable (numpy) host buffers.  L2 flushed before each step."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2005_01182_b200 import Solver, workloads as W

B, N = 4096, 128
c = W.CONFIGS["c3"].make()
s = Solver(0)
st = torch.cuda.current_stream()
s.set_stream(st.cuda_stream)
dc = torch.from_numpy(c).cuda()
r2c = torch.empty((B, N), dtype=torch.int32, device="cuda")
u = torch.empty((B, N), dtype=torch.int64, device="cuda"); v = torch.empty_like(u)
tot = torch.empty(B, dtype=torch.int64, device="cuda"); status = torch.empty(B, dtype=torch.int32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")


def timed(call, steps=20):
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    ts = []
    for k in range(steps):
        flush.fill_(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); call(); e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


out = {}
out["async_ms"] = timed(lambda: s.solve_batch_async(dc, B, N, 1, r2c, u, v, tot, status))
out["tot_fnv"] = W.fnv1a64(tot.cpu().numpy())
hc = torch.from_numpy(c).pin_memory()
hr = [torch.empty((B, N), dtype=torch.int32).pin_memory(), torch.empty((B, N), dtype=torch.int64).pin_memory(),
      torch.empty((B, N), dtype=torch.int64).pin_memory(), torch.empty(B, dtype=torch.int64).pin_memory()]
out["e2e_pinned_ms"] = timed(lambda: s.solve_batch_into(hc, B, N, 1, *hr, stats=False), 10)
pg = [np.empty((B, N), np.int32), np.empty((B, N), np.int64), np.empty((B, N), np.int64), np.empty(B, np.int64)]
out["e2e_pageable_ms"] = timed(lambda: s.solve_batch_into(c, B, N, 1, *pg, stats=False), 10)
out["pageable_matches"] = bool(np.array_equal(pg[3], hr[3].numpy()) and np.array_equal(pg[1], hr[1].numpy())
                               and np.array_equal(pg[0], hr[0].numpy()))
print(json.dumps(out))
