"""Worker for tests/test_sharded.py (spawned once per rank)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def make_cases():
    from paper_2005_01182_b200 import workloads as W
    rng = np.random.default_rng(42)
    cases = []
    for t in range(12):
        n = int(rng.integers(1, 70))
        hi = int(rng.choice([1, 3, 100, 10**6]))
        cases.append(rng.integers(0, hi + 1, size=(n, n)).astype(np.int32))
    cases.append(W.CONFIGS["c1"].make())
    return cases


def run(rank, world, port, mode, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2005_01182_b200.sharded import GroupExchange, column_span
    results = []
    if mode == "sim":
        lib = C.CDLL(os.path.join(ROOT, "tests", "cpp", "build", "libshardsim.so"))
        ex = GroupExchange()
        for c in make_cases():
            n = c.shape[0]
            for seed in (1, 0):
                cb, nc = column_span(n, world, rank)
                slab = np.ascontiguousarray(c[:, cb:cb + nc])
                r2c = np.full(n, -1, np.int32)
                u = np.zeros(n, np.int64)
                v = np.zeros(max(nc, 1), np.int64)
                out = np.zeros(4, np.int64)
                rc = lib.shardsim_solve(C.c_void_p(slab.ctypes.data), C.c_int32(n), C.c_int64(max(nc, 1)),
                                        C.c_int32(cb), C.c_int32(nc), C.c_int32(seed), C.c_int32(world),
                                        C.c_int32(rank), ex.ar, ex.ag, C.c_void_p(r2c.ctypes.data),
                                        C.c_void_p(u.ctypes.data), C.c_void_p(v.ctypes.data),
                                        C.c_void_p(out.ctypes.data))
                results.append((rc, r2c, u, v[:nc], int(out[0]), int(out[1]), cb))
    elif mode.startswith("fail"):  # "fail:<op>:<at>": rank 1 fails, every rank must return -1
        _, op, at = mode.split(":")
        lib = C.CDLL(os.path.join(ROOT, "tests", "cpp", "build", "libshardsim.so"))
        ex = GroupExchange()
        c = make_cases()[-1]  # config 1, n = 256
        n = c.shape[0]
        cb, nc = column_span(n, world, rank)
        slab = np.ascontiguousarray(c[:, cb:cb + nc])
        r2c = np.full(n, -1, np.int32)
        u = np.zeros(n, np.int64)
        v = np.zeros(max(nc, 1), np.int64)
        out = np.zeros(4, np.int64)
        rc = lib.shardsim_solve_fail(
            C.c_void_p(slab.ctypes.data), C.c_int32(n), C.c_int64(max(nc, 1)), C.c_int32(cb),
            C.c_int32(nc), C.c_int32(1), C.c_int32(world), C.c_int32(rank), ex.ar, ex.ag,
            C.c_void_p(r2c.ctypes.data), C.c_void_p(u.ctypes.data), C.c_void_p(v.ctypes.data),
            C.c_void_p(out.ctypes.data), C.c_int32(int(op) if rank == 1 else 0), C.c_int32(int(at)))
        results.append(rc)
    elif mode == "dev":  # the device-exchange protocol through the Python helpers (one rank)
        from paper_2005_01182_b200 import Solver
        from paper_2005_01182_b200.sharded import init_exchange, open_device_exchange, solve_sharded_device
        s = Solver(0)
        init_exchange(s, "group")
        for c in make_cases():
            n = c.shape[0]
            cols = open_device_exchange(s, n)
            for seed in (1, 0):
                cb = rank * cols
                nc = max(0, min(cols, n - cb))
                slab = np.ascontiguousarray(c[:, cb:cb + nc])
                r2c, u, v, tot, st = solve_sharded_device(s, slab, n, cb, seed)
                results.append((0, r2c, u, v, tot, st["dual_steps"], cb))
    else:  # "gpu"/"nccl": the CUDA slab kernels; exchange through this gloo group
        # (ranks share cuda:0) or through NCCL (one rank per GPU)
        from paper_2005_01182_b200 import Solver
        from paper_2005_01182_b200.sharded import init_exchange, solve_sharded
        s = Solver(0)
        init_exchange(s, "group" if mode == "gpu" else "nccl")
        for c in make_cases():
            n = c.shape[0]
            for seed in (1, 0):
                cb, nc = column_span(n, world, rank)
                slab = np.ascontiguousarray(c[:, cb:cb + nc])
                r2c, u, v, tot, st = solve_sharded(s, slab, n, cb, seed)
                results.append((0, r2c, u, v, tot, st["dual_steps"], cb))
    np.save(os.path.join(outdir, f"rank{rank}.npy"), np.array(results, dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()
