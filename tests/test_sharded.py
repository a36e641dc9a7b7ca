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
