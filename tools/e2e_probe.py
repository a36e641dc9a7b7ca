"""End-to-end (host buffers) batch solve time by pipeline chunk schedule
(KMB_OPT_PIPELINE) and shard size, beside the bare pinned H2D of the same bytes.

    python tools/e2e_probe.py [--sizes 4096,2048,1024,512] [--opts 0,8,16,-16]
"""
import argparse
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import _gen_c3  # noqa: E402
from paper_2005_01182_b200 import Solver  # noqa: E402
from paper_2005_01182_b200.api import OPT_PIPELINE  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="4096,2048,1024,512")
ap.add_argument("--opts", default="0,8,16,32,-4,-16")
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
N = 128
host_all = _gen_c3(0, 4096)
s = Solver(0)
stream = torch.cuda.current_stream()
s.set_stream(stream.cuda_stream)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")


def timed(fn, steps):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(steps):
        flush.fill_(k)
        ev[k][0].record(stream)
        fn()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


for b in [int(x) for x in args.sizes.split(",")]:
    host = torch.from_numpy(np.ascontiguousarray(host_all[:b])).pin_memory()
    d = host.cuda()
    r2c = torch.empty((b, N), dtype=torch.int32, device="cuda")
    du = torch.empty((b, N), dtype=torch.int64, device="cuda")
    dv = torch.empty((b, N), dtype=torch.int64, device="cuda")
    dt = torch.empty(b, dtype=torch.int64, device="cuda")
    hr = torch.empty((b, N), dtype=torch.int32).pin_memory()
    hu = torch.empty((b, N), dtype=torch.int64).pin_memory()
    hv = torch.empty((b, N), dtype=torch.int64).pin_memory()
    ht = torch.empty(b, dtype=torch.int64).pin_memory()
    dev_ms = timed(lambda: s.solve_batch_into(d, b, N, 1, r2c, du, dv, dt, stats=False), args.steps)
    h2d_ms = timed(lambda: d.copy_(host, non_blocking=True), args.steps)
    print(f"batch {b}: device {dev_ms:.3f} ms, bare H2D {h2d_ms:.3f} ms "
          f"({host.numel() * 4 / h2d_ms / 1e6:.1f} GB/s)", flush=True)
    for o in [int(x) for x in args.opts.split(",")]:
        s.set_option(OPT_PIPELINE, o)
        for _ in range(3):
            s.solve_batch_into(host, b, N, 1, hr, hu, hv, ht, stats=False)
        ms = timed(lambda: s.solve_batch_into(host, b, N, 1, hr, hu, hv, ht, stats=False), args.steps)
        torch.cuda.synchronize()
        ok = torch.equal(hr, r2c.cpu()) and torch.equal(hu, du.cpu()) and torch.equal(ht, dt.cpu())
        print(f"  pipeline {o:4d}: e2e {ms:.3f} ms = {b / ms * 1e3:,.0f} solves/s "
              f"(over H2D {ms - h2d_ms:+.3f} ms) ok={ok}", flush=True)
    s.set_option(OPT_PIPELINE, 0)
