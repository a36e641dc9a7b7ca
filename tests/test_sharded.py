"""Column-sharded single-instance protocol (config 5's multi-GPU mode) with
world_size 2 and 3 over torch.distributed gloo:

* CPU: the product's protocol (csrc/kmb_shard_proto.h) instantiated with
  simulated CPU shards (tests/cpp/shard_sim.cpp) — exchange logic end to end;
* GPU: the real CUDA slab kernels (kmb_solve_sharded_i32), two ranks sharing
  cuda:0 (no kernel waits on another rank: every exchange is host-driven).

Both against the unmodified reference: total cost, u, and the concatenated
per-rank v bit-exact; the dual-step count equals the restatement's.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from tests import _shard_worker as W


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, mode):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(W.run, args=(world, _port(), mode, d), nprocs=world, join=True)
        return [np.load(os.path.join(d, f"rank{r}.npy"), allow_pickle=True) for r in range(world)]


def _check(per_rank):
    cases = W.make_cases()
    k = 0
    for c in cases:
        for seed in (1, 0):
            ref = O.ref_solve_batched_km(c) if seed == 1 else O.ref_solve_km(c)
            outs = [pr[k] for pr in per_rank]
            k += 1
            for rc, r2c, u, v, tot, ds, cb in outs:
                assert rc == 0
                assert tot == ref.total_cost
                np.testing.assert_array_equal(u, ref.u)
                assert sorted(r2c.tolist()) == list(range(c.shape[0]))
            vfull = np.concatenate([o[3] for o in sorted(outs, key=lambda o: o[6])])
            np.testing.assert_array_equal(vfull, ref.v)
            if seed == 1:
                assert outs[0][5] == O.kmo_solve_batched(c).dual_steps


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_protocol_cpu_gloo(world):
    _check(_run(world, "sim"))


@pytest.mark.timeout(120)
@pytest.mark.parametrize("op,at", [(8, 1), (2, 7), (3, 5), (5, 3), (7, 1)])
def test_sharded_local_failure_fails_every_rank(op, at):
    """A failure on one rank (before the protocol, or in any slab operation at
    any round) is voted on at the next collective: every rank returns -1
    instead of the others waiting forever."""
    per_rank = _run(2, f"fail:{op}:{at}")
    assert [int(r[0]) for r in per_rank] == [-1, -1]


@pytest.mark.gpu
def test_sharded_cuda_two_ranks_one_gpu():
    _check(_run(2, "gpu"))


@pytest.mark.gpu
def test_sharded_cuda_nccl_world1():
    """The NCCL exchange path (ncclAllReduce ncclMin / ncclAllGather) on the one
    GPU a test box has: a single-rank communicator."""
    _check(_run(1, "nccl"))


# ---- device-side exchange (k_solve_sharded, kmb_shard_dev.cu) ------------------

@pytest.mark.gpu
@pytest.mark.parametrize("ranks", [1, 2, 3, 4, 8])
def test_sharded_device_exchange_local(solver, ranks):
    """The device-exchange column-sharded engine with `ranks` ranks as CTA
    groups of one launch: duals and total bit-exact against the reference, the
    matching equal to the single-GPU grid engine's (both deterministic), every
    replica of the row side identical (checked inside the call)."""
    from paper_2005_01182_b200 import KMB_SEED_BATCHED, KMB_SEED_KM
    from paper_2005_01182_b200.api import OPT_ENGINE
    for c in W.make_cases():
        for seed in (KMB_SEED_BATCHED, KMB_SEED_KM):
            ref = O.ref_solve_batched_km(c) if seed == KMB_SEED_BATCHED else O.ref_solve_km(c)
            r = solver.solve_sharded_local(c, ranks, seed)
            assert r.stats["engine"] == 10
            assert r.total_cost == ref.total_cost
            np.testing.assert_array_equal(r.u, ref.u)
            np.testing.assert_array_equal(r.v, ref.v)
            solver.set_option(OPT_ENGINE, 1)
            g = solver.solve(c, seed)
            solver.set_option(OPT_ENGINE, 0)
            np.testing.assert_array_equal(r.row_to_col, g.row_to_col)
            assert r.stats["dual_steps"] == g.stats["dual_steps"]


@pytest.mark.gpu
@pytest.mark.parametrize("ranks", [2, 4])
def test_sharded_device_exchange_config5(solver, ranks):
    """Config 5 (n = 16384, 1 GiB) column-sharded with the exchange on the
    device: total cost and the FNV-1a hashes of u and v equal the committed
    reference golden."""
    import json
    from paper_2005_01182_b200 import workloads as Wk
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "configs.json")))["c5"]
    c = Wk.CONFIGS["c5"].make()
    r = solver.solve_sharded_local(c, ranks)
    assert r.total_cost == g["total_cost"]
    assert Wk.fnv1a64(r.u) == g["u_fnv"] and Wk.fnv1a64(r.v) == g["v_fnv"]


@pytest.mark.gpu
def test_sharded_device_exchange_gpu_rank_path_world1(solver):
    """The GPU-rank entry points (kmb_shard_dev_open / _connect /
    kmb_solve_sharded_dev_i32) on the one GPU of a test box: a single rank, its
    IPC handle produced, no peer to map."""
    import ctypes as C
    from paper_2005_01182_b200.api import Stats
    lib = solver._lib
    for c in W.make_cases()[:6] + [W.make_cases()[-1]]:
        n = c.shape[0]
        cols = C.c_int32()
        handle = (C.c_uint8 * 64)()
        solver._check(lib.kmb_shard_dev_open(solver._h, n, 1, 0, C.byref(cols), handle))
        assert cols.value >= n
        solver._check(lib.kmb_shard_dev_connect(solver._h, handle))
        r2c = np.full(n, -1, np.int32)
        u = np.zeros(n, np.int64)
        v = np.zeros(n, np.int64)
        tot = C.c_int64()
        st = Stats()
        cc = np.ascontiguousarray(c)
        solver._check(lib.kmb_solve_sharded_dev_i32(
            solver._h, C.c_void_p(cc.ctypes.data), n, n, 0, n, 1, C.c_void_p(r2c.ctypes.data),
            C.c_void_p(u.ctypes.data), C.c_void_p(v.ctypes.data), C.byref(tot), C.byref(st)))
        ref = O.ref_solve_batched_km(c)
        assert tot.value == ref.total_cost
        np.testing.assert_array_equal(u, ref.u)
        np.testing.assert_array_equal(v, ref.v)


@pytest.mark.gpu
def test_sharded_device_exchange_python_helpers_world1():
    """sharded.open_device_exchange / solve_sharded_device under
    torch.distributed (IPC handle allgather, host barriers through the group)
    with the one rank a test box's GPU can hold: the device-exchange kernels of
    several ranks must not share a GPU as separate launches."""
    _check(_run(1, "dev"))


@pytest.mark.gpu
def test_sharded_device_exchange_errors(solver):
    c = np.ones((9, 9), np.int32)
    c[4, 4] = -1
    from paper_2005_01182_b200 import KmbError
    with pytest.raises(KmbError, match="costs must be nonnegative"):
        solver.solve_sharded_local(c, 2)
    c[4, 4] = 2**29
    with pytest.raises(KmbError, match="device range"):
        solver.solve_sharded_local(c, 2)
    with pytest.raises(KmbError, match="bad arguments"):
        solver.solve_sharded_local(np.ones((3, 3), np.int32), 9)
