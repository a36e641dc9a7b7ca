"""Auction throughput: GPU (kmb_auction_i32, device-resident costs) vs the
reference auction on the host (oracle/_ref, one instance per thread)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.api import AuctionConfig
s = Solver(0)
for key in os.environ.get("CFGS", "c3,c1,c2").split(","):
    c = W.CONFIGS[key].make()
    if c.ndim == 2: c = c[None]
    b, n, _ = c.shape
    dc = torch.from_numpy(c).cuda()
    pr = torch.empty((b, n), dtype=torch.float64, device="cuda"); r2c = torch.empty((b, n), dtype=torch.int32, device="cuda")
    tot = torch.empty(b, dtype=torch.int64, device="cuda"); bids = torch.empty(b, dtype=torch.int64, device="cuda")
    for scaled, eps in [(1, 0.0), (0, 1.0)]:
        if key == "c2" and not scaled: continue
        cfg = AuctionConfig(scaled, eps, 4.0, 0.0, 10**9, 0.0)
        ts = [s.auction_into(dc, b, n, cfg, pr, r2c, tot, bids) for _ in range(3 if b > 1 else 2)]
        t = min(ts)
        # reference on the host: a bounded sample
        k = min(b, 64)
        t0 = time.perf_counter()
        nb = 0
        for i in range(k):
            r = O.ref_solve_auction_scaled(c[i]) if scaled else O.ref_solve_auction(c[i], eps)
            nb += r.iterations
            assert r.iterations == int(bids[i]) and r.total_cost == int(tot[i])
        tc = (time.perf_counter() - t0) / k
        print(json.dumps({"cfg": key, "scaled": scaled, "batch": b, "n": n, "gpu_ms": t * 1e3,
                          "gpu_solves_per_s": b / t, "bids_mean": float(bids.double().mean()),
                          "gpu_ns_per_bid_per_instance": t / float(bids.double().max()) * 1e9,
                          "ref_ms_per_solve_1thread": tc * 1e3, "speedup_vs_1thread": tc * b / t}), flush=True)
