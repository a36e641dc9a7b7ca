"""Column-sharded single-instance solve across ranks (BASELINE config 5's
multi-GPU mode; C ABI ``kmb_solve_sharded_i32``, protocol in
``csrc/kmb_shard_proto.h``).

Rank r of a torch.distributed job owns columns ``[r*n/N, (r+1)*n/N)``.  The
per-round min-slack combine and the entry exchanges run either

* over NCCL (``exchange="nccl"``): rank 0 creates an NCCL unique id, it is
  broadcast through the process group, and the library drives
  ``ncclAllReduce(ncclMin)`` / ``ncclAllGather`` on its own communicator, or
* through the process group itself (``exchange="group"``): the library calls
  back into Python, which issues ``all_reduce(MIN)`` / ``all_gather`` on CPU
  tensors — any backend, e.g. gloo, and ranks may share a GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .api import Stats, Solver, _stats_dict

ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_int64), C.c_int32, C.c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)


def column_span(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous column shard of rank `rank`: (col_begin, ncols)."""
    per, extra = divmod(n, world)
    begin = rank * per + min(rank, extra)
    return begin, per + (1 if rank < extra else 0)


class GroupExchange:
    """ctypes callbacks running the collectives on a torch.distributed group."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self._torch, self._dist, self._group = torch, dist, group
        self.world = dist.get_world_size(group)

        def allreduce_min(ptr, count, _user):
            try:
                buf = np.ctypeslib.as_array(ptr, shape=(count,))
                t = torch.from_numpy(buf.copy())
                dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
                buf[:] = t.numpy()
                return 0
            except Exception:  # surfaced as a KmbError by the library
                return -1

        def allgather(send, nbytes, recv, _user):
            try:
                src = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), shape=(nbytes,))
                t = torch.from_numpy(src.copy())
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.world)]
                dist.all_gather(outs, t, group=group)
                dst = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)),
                                            shape=(nbytes * self.world,))
                dst[:] = torch.cat(outs).numpy()
                return 0
            except Exception:
                return -1

        self.ar = ALLREDUCE_FN(allreduce_min)  # keep references alive
        self.ag = ALLGATHER_FN(allgather)


def init_exchange(solver: Solver, exchange: str = "group", group=None):
    """Attach the rank's collective to the solver context."""
    import torch
    import torch.distributed as dist
    lib = solver._lib
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if exchange == "nccl":
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            solver._check(lib.kmb_nccl_unique_id(uid))
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
        dist.broadcast(t, src=0, group=group)
        uid = (C.c_uint8 * 128)(*t.tolist())
        solver._check(lib.kmb_shard_init_nccl(solver._h, world, rank, uid))
        solver._exchange = None
    elif exchange == "group":
        ex = GroupExchange(group)
        solver._check(lib.kmb_shard_init_callbacks(solver._h, world, rank, ex.ar, ex.ag, None))
        solver._exchange = ex
    else:
        raise ValueError(exchange)


def solve_sharded(solver: Solver, slab: np.ndarray, n: int, col_begin: int, seed: int = 1):
    """Collective: every rank passes its n x ncols column slab (host or device
    array).  Returns (row_to_col[n], u[n], v_slab[ncols], total_cost, stats)."""
    lib = solver._lib
    s = np.ascontiguousarray(slab, dtype=np.int32) if isinstance(slab, np.ndarray) else slab
    ncols = s.shape[1]
    r2c = np.full(n, -1, np.int32)
    u = np.zeros(n, np.int64)
    v = np.zeros(max(ncols, 1), np.int64)
    tot = C.c_int64()
    st = Stats()
    ptr = s.ctypes.data if isinstance(s, np.ndarray) else s.data_ptr()
    rc = lib.kmb_solve_sharded_i32(solver._h, C.c_void_p(ptr), n, ncols, col_begin, ncols, seed,
                                   r2c.ctypes.data_as(C.c_void_p), u.ctypes.data_as(C.c_void_p),
                                   v.ctypes.data_as(C.c_void_p), C.byref(tot), C.byref(st))
    solver._check(rc)
    return r2c, u, v[:ncols], tot.value, _stats_dict(st)


# ---- device-side exchange (kmb_shard_dev_*, csrc/kmb_shard_dev.cu) --------------

def open_device_exchange(solver: Solver, n: int, group=None) -> int:
    """Collective setup of the device-exchange protocol for an n x n instance:
    each rank allocates its window, the 64-byte CUDA IPC handles are allgathered
    through the process group and every rank maps its peers' windows.  Needs
    ``init_exchange`` too (two host barriers per solve).  Returns slab_cols:
    rank r holds columns [r * slab_cols, min(n, (r + 1) * slab_cols))."""
    import torch
    import torch.distributed as dist
    lib = solver._lib
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    cols = C.c_int32()
    mine = (C.c_uint8 * 64)()
    solver._check(lib.kmb_shard_dev_open(solver._h, n, world, rank, C.byref(cols), mine))
    outs = [torch.empty(64, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(outs, torch.tensor(list(bytes(mine)), dtype=torch.uint8), group=group)
    allh = (C.c_uint8 * (64 * world))(*torch.cat(outs).tolist())
    solver._check(lib.kmb_shard_dev_connect(solver._h, allh))
    return cols.value


def solve_sharded_device(solver: Solver, slab, n: int, col_begin: int, seed: int = 1):
    """Collective solve with the exchange on the device (after
    ``open_device_exchange``): every rank passes its n x ncols column slab
    (host or device array).  Returns (row_to_col[n], u[n], v_slab[ncols],
    total_cost, stats)."""
    lib = solver._lib
    s = np.ascontiguousarray(slab, dtype=np.int32) if isinstance(slab, np.ndarray) else slab
    ncols = s.shape[1]
    r2c = np.full(n, -1, np.int32)
    u = np.zeros(n, np.int64)
    v = np.zeros(max(ncols, 1), np.int64)
    tot = C.c_int64()
    st = Stats()
    ptr = s.ctypes.data if isinstance(s, np.ndarray) else s.data_ptr()
    rc = lib.kmb_solve_sharded_dev_i32(solver._h, C.c_void_p(ptr), n, ncols, col_begin, ncols, seed,
                                       r2c.ctypes.data_as(C.c_void_p), u.ctypes.data_as(C.c_void_p),
                                       v.ctypes.data_as(C.c_void_p), C.byref(tot), C.byref(st))
    solver._check(rc)
    return r2c, u, v[:ncols], tot.value, _stats_dict(st)
