"""Python host mirror of the reference's solver entry points over the C ABI.

``solve_km`` / ``solve_batched_km`` follow ``ot::solve_km`` (hungarian.cpp:55-136)
and ``ot::solve_batched_km`` (hungarian.cpp:313-381): cost matrix in; assignment,
total cost and row/column duals out; the same exceptions with the same
messages (``ValueError`` standing in for ``std::invalid_argument``).  The C++
mirror with the reference's exact types is ``include/kmb_ot.hpp``; this module is
what the tests and ``bench.py`` use.

Every call goes through ``libkmb.so`` (CUDA, sm_100a).  There is no CPU path:
if the library or a B200 is missing the call raises ``KmbUnavailable``.
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _build

KMB_SEED_KM = 0
KMB_SEED_BATCHED = 1
KMB_OK, KMB_EINVAL, KMB_ENEGATIVE, KMB_ERANGE = 0, 1, 2, 3  # include/kmb.h status codes
OPT_MAX_CTAS, OPT_ENGINE, OPT_WARPS_PER_SM, OPT_PIPELINE, OPT_RESIDENT16 = 1, 3, 4, 6, 7

# every symbol include/kmb.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = ("kmb_create", "kmb_destroy", "kmb_set_stream", "kmb_set_option", "kmb_solve_i32",
               "kmb_solve_batch_i32", "kmb_solve_batch_async_i32", "kmb_solve_batch_multi_i32",
               "kmb_nccl_unique_id",
               "kmb_shard_init_nccl",
               "kmb_shard_init_callbacks", "kmb_solve_sharded_i32", "kmb_bench_scan",
               "kmb_last_instance_stats", "kmb_costs_from_points", "kmb_auction_i32",
               "kmb_solve_i64", "kmb_solve_batch_i64", "kmb_quantize_i64",
               "kmb_solve_batched_km_i64", "kmb_shard_dev_open", "kmb_shard_dev_connect",
               "kmb_solve_sharded_dev_i32", "kmb_solve_sharded_local_i32",
               "kmb_last_error", "kmb_abi_version")


class KmbUnavailable(RuntimeError):
    """The CUDA library or an sm_100 device is missing — no fallback exists."""


class KmbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class Stats(C.Structure):
    _fields_ = [("phases", C.c_int64), ("dual_steps", C.c_int64), ("rows_scanned", C.c_int64),
                ("cost_bytes_read", C.c_int64), ("seconds", C.c_double),
                ("converged", C.c_int32), ("engine", C.c_int32), ("rounds", C.c_int64),
                ("stage_ns", C.c_int64 * 6), ("max_instance_cycles", C.c_int64),
                ("sum_instance_cycles", C.c_int64), ("segment_rows", C.c_int64)]


class AuctionConfig(C.Structure):
    """``kmb_auction_config`` (include/kmb.h)."""
    _fields_ = [("scaled", C.c_int32), ("epsilon", C.c_double), ("theta", C.c_double),
                ("epsilon_final", C.c_double), ("max_bids", C.c_int64),
                ("time_budget_s", C.c_double)]


_lib = None


def load_library(path: str | None = None):
    """Load libkmb.so (built in-tree by ``_build.build_lib``).  Fails loudly."""
    global _lib
    if _lib is None:
        path = path or os.environ.get("KMB_LIB") or _build.LIB_SO
        if not os.path.exists(path):
            raise KmbUnavailable(f"{path} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
        lib = C.CDLL(path)
        vp = C.c_void_p
        lib.kmb_create.argtypes = [C.c_int, C.POINTER(vp)]
        lib.kmb_destroy.argtypes = [vp]
        lib.kmb_destroy.restype = None
        lib.kmb_set_stream.argtypes = [vp, vp]
        lib.kmb_set_option.argtypes = [vp, C.c_int, C.c_int64]
        lib.kmb_solve_i32.argtypes = [vp, vp, C.c_int32, C.c_int64, C.c_int32, C.c_double,
                                      vp, vp, vp, vp, C.POINTER(Stats)]
        lib.kmb_solve_batch_i32.argtypes = [vp, vp, C.c_int32, C.c_int32, C.c_int32,
                                            vp, vp, vp, vp, C.POINTER(Stats)]
        lib.kmb_solve_batch_async_i32.argtypes = [vp, vp, C.c_int32, C.c_int32, C.c_int32,
                                                  vp, vp, vp, vp, vp]
        lib.kmb_solve_batch_multi_i32.argtypes = [C.POINTER(vp), C.c_int32, vp, C.c_int32, C.c_int32,
                                                  C.c_int32, vp, vp, vp, vp, C.POINTER(Stats)]
        lib.kmb_bench_scan.argtypes = [vp, vp, C.c_int32, C.c_int64, C.c_int32,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.kmb_costs_from_points.argtypes = [vp, vp, vp, C.c_int32, C.c_int32, C.c_int32,
                                              C.c_int32, C.c_int32, C.c_double, C.c_int32, vp]
        lib.kmb_auction_i32.argtypes = [vp, vp, C.c_int32, C.c_int32, C.POINTER(AuctionConfig),
                                        vp, vp, vp, vp, vp, vp, C.POINTER(C.c_double)]
        lib.kmb_solve_i64.argtypes = lib.kmb_solve_i32.argtypes
        lib.kmb_solve_batch_i64.argtypes = lib.kmb_solve_batch_i32.argtypes
        lib.kmb_quantize_i64.argtypes = [vp, vp, C.c_int64, C.c_int64, vp, C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int32)]
        lib.kmb_solve_batched_km_i64.argtypes = [vp, vp, C.c_int32, C.c_int64, C.c_double, vp, vp, vp,
                                                 vp, vp, C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                                 C.POINTER(Stats)]
        lib.kmb_shard_dev_open.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32), vp]
        lib.kmb_shard_dev_connect.argtypes = [vp, vp]
        lib.kmb_solve_sharded_dev_i32.argtypes = [vp, vp, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                                  C.c_int32, vp, vp, vp, vp, C.POINTER(Stats)]
        lib.kmb_solve_sharded_local_i32.argtypes = [vp, vp, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                                    vp, vp, vp, vp, C.POINTER(Stats)]
        lib.kmb_last_error.restype = C.c_char_p
        lib.kmb_abi_version.restype = C.c_int
        _lib = lib
    return _lib


def _ptr(a) -> int | None:
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch tensor (host or device)
        return a.data_ptr()
    return a.ctypes.data


@dataclass
class Result:
    """Mirror of ``ot::SolveResult`` (core.hpp:90-98) + DualPotentials + Matching."""
    row_to_col: object
    u: object
    v: object
    total_cost: object
    iterations: int = 0
    exact: bool = True
    converged: bool = True
    wall_seconds: float = 0.0
    stats: dict = field(default_factory=dict)
    prices: object = None  # auction: final column prices

    @property
    def objective(self) -> float:
        return float(self.total_cost)


class Solver:
    """One device context (workspace cached across calls)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        lib = load_library()
        self._lib = lib
        h = C.c_void_p()
        rc = lib.kmb_create(device, C.byref(h))
        if rc != 0:
            raise KmbUnavailable(lib.kmb_last_error().decode())
        self._h = h
        if stream is not None:
            self.set_stream(stream)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.kmb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream: int):
        self._check(self._lib.kmb_set_stream(self._h, C.c_void_p(stream)))

    def set_option(self, option: int, value: int):
        self._check(self._lib.kmb_set_option(self._h, option, int(value)))

    def _check(self, rc: int):
        if rc != 0:
            msg = self._lib.kmb_last_error().decode()
            if rc > 0:
                raise KmbError(rc, msg)
            raise KmbError(rc, msg)

    # -- raw C-ABI calls -------------------------------------------------------
    def solve_into(self, cost, n: int, ld: int, seed: int, row_to_col, u, v, total_cost,
                   time_budget_s: float = 0.0, stats: bool = True) -> Stats | None:
        st = Stats() if stats else None
        rc = self._lib.kmb_solve_i32(self._h, C.c_void_p(_ptr(cost)), n, ld, seed, time_budget_s,
                                     C.c_void_p(_ptr(row_to_col)), C.c_void_p(_ptr(u)),
                                     C.c_void_p(_ptr(v)), C.c_void_p(_ptr(total_cost)),
                                     C.byref(st) if st is not None else None)
        self._check(rc)
        return st

    def solve_batch_into(self, costs, batch: int, n: int, seed: int, row_to_col, u, v,
                         total_cost, stats: bool = True) -> Stats | None:
        st = Stats() if stats else None
        rc = self._lib.kmb_solve_batch_i32(self._h, C.c_void_p(_ptr(costs)), batch, n, seed,
                                           C.c_void_p(_ptr(row_to_col)), C.c_void_p(_ptr(u)),
                                           C.c_void_p(_ptr(v)), C.c_void_p(_ptr(total_cost)),
                                           C.byref(st) if st is not None else None)
        self._check(rc)
        return st

    def solve_i64_into(self, cost, n: int, ld: int, seed: int, row_to_col, u, v, total_cost,
                       time_budget_s: float = 0.0, stats: bool = True) -> Stats | None:
        """``kmb_solve_i64``: int64 costs over the reference's whole range."""
        st = Stats() if stats else None
        rc = self._lib.kmb_solve_i64(self._h, C.c_void_p(_ptr(cost)), n, ld, seed, time_budget_s,
                                     C.c_void_p(_ptr(row_to_col)), C.c_void_p(_ptr(u)),
                                     C.c_void_p(_ptr(v)), C.c_void_p(_ptr(total_cost)),
                                     C.byref(st) if st is not None else None)
        self._check(rc)
        return st

    def solve_batch_i64_into(self, costs, batch: int, n: int, seed: int, row_to_col, u, v,
                             total_cost, stats: bool = True) -> Stats | None:
        st = Stats() if stats else None
        rc = self._lib.kmb_solve_batch_i64(self._h, C.c_void_p(_ptr(costs)), batch, n, seed,
                                           C.c_void_p(_ptr(row_to_col)), C.c_void_p(_ptr(u)),
                                           C.c_void_p(_ptr(v)), C.c_void_p(_ptr(total_cost)),
                                           C.byref(st) if st is not None else None)
        self._check(rc)
        return st

    def quantize(self, cost, B: int, chat=None) -> tuple[int, bool]:
        """``kmb_quantize_i64`` (K11 on the device): fills ``chat`` (optional,
        same size as ``cost``) and returns (N, lossless)."""
        N = C.c_int64()
        ll = C.c_int32()
        count = int(np.prod(cost.shape)) if len(cost.shape) else 1
        self._check(self._lib.kmb_quantize_i64(self._h, C.c_void_p(_ptr(cost)), count, int(B),
                                               C.c_void_p(_ptr(chat)), C.byref(N), C.byref(ll)))
        return int(N.value), bool(ll.value)

    def solve_batched_km_into(self, cost, n: int, B: int, row_to_col, u, v, total_cost,
                              chat=None, time_budget_s: float = 0.0) -> tuple[Stats, int, bool]:
        """``kmb_solve_batched_km_i64``: the reference's solve_batched_km on the
        device (quantization included); returns (stats, N, lossless)."""
        st = Stats()
        N = C.c_int64()
        ll = C.c_int32()
        self._check(self._lib.kmb_solve_batched_km_i64(
            self._h, C.c_void_p(_ptr(cost)), n, int(B), time_budget_s, C.c_void_p(_ptr(row_to_col)),
            C.c_void_p(_ptr(u)), C.c_void_p(_ptr(v)), C.c_void_p(_ptr(total_cost)),
            C.c_void_p(_ptr(chat)), C.byref(N), C.byref(ll), C.byref(st)))
        return st, int(N.value), bool(ll.value)

    def solve_sharded_local(self, cost, nranks: int, seed: int = KMB_SEED_BATCHED):
        """``kmb_solve_sharded_local_i32``: the device-exchange column-sharded
        engine with ``nranks`` ranks as CTA groups of one launch on this GPU
        (replicas checked equal after the solve).  numpy or torch input."""
        n = cost.shape[0]
        r2c = np.full(n, -1, np.int32)
        u = np.zeros(n, np.int64)
        v = np.zeros(n, np.int64)
        tot = np.zeros(1, np.int64)
        st = Stats()
        if not hasattr(cost, "data_ptr"):
            cost = np.ascontiguousarray(cost, dtype=np.int32)
        self._check(self._lib.kmb_solve_sharded_local_i32(
            self._h, C.c_void_p(_ptr(cost)), n, n, nranks, seed, C.c_void_p(r2c.ctypes.data),
            C.c_void_p(u.ctypes.data), C.c_void_p(v.ctypes.data), C.c_void_p(tot.ctypes.data),
            C.byref(st)))
        return Result(r2c, u, v, int(tot[0]), iterations=int(st.phases + st.dual_steps),
                      stats=_stats_dict(st))

    def solve_batch_async(self, costs, batch: int, n: int, seed: int, row_to_col, u, v,
                          total_cost, status) -> None:
        """Stream-ordered batch solve (kmb_solve_batch_async_i32): device buffers
        only; enqueues on the solver's stream and returns without waiting;
        per-instance statuses land in ``status`` (device int32)."""
        self._check(self._lib.kmb_solve_batch_async_i32(
            self._h, C.c_void_p(_ptr(costs)), batch, n, seed, C.c_void_p(_ptr(row_to_col)),
            C.c_void_p(_ptr(u)), C.c_void_p(_ptr(v)), C.c_void_p(_ptr(total_cost)),
            C.c_void_p(_ptr(status))))

    def last_instance_stats(self, batch: int):
        """Per-instance counters of the last batch solve: (batch, 11) int64."""
        out = np.zeros(batch * 11, np.int64)
        cnt = C.c_int64()
        self._check(self._lib.kmb_last_instance_stats(self._h, C.c_void_p(out.ctypes.data), out.size,
                                                      C.byref(cnt)))
        return out.reshape(batch, 11)

    def bench_scan(self, cost, n: int, ld: int, iters: int = 5) -> tuple[float, float]:
        """Full-frontier scan microbenchmark: (seconds per pass, GB/s)."""
        t = C.c_double()
        g = C.c_double()
        self._check(self._lib.kmb_bench_scan(self._h, C.c_void_p(_ptr(cost)), n, ld, iters,
                                             C.byref(t), C.byref(g)))
        return t.value, g.value

    def auction_into(self, costs, batch: int, n: int, cfg: AuctionConfig, prices=None,
                     row_to_col=None, total_cost=None, bids=None, converged=None,
                     epsilon_last=None) -> float:
        """Raw ``kmb_auction_i32``; returns the device seconds."""
        sec = C.c_double()
        self._check(self._lib.kmb_auction_i32(
            self._h, C.c_void_p(_ptr(costs)), batch, n, C.byref(cfg), C.c_void_p(_ptr(prices)),
            C.c_void_p(_ptr(row_to_col)), C.c_void_p(_ptr(total_cost)), C.c_void_p(_ptr(bids)),
            C.c_void_p(_ptr(converged)), C.c_void_p(_ptr(epsilon_last)), C.byref(sec)))
        return sec.value

    def auction(self, costs, scaled: bool = True, epsilon: float = 0.0, theta: float = 4.0,
                epsilon_final: float = 0.0, max_bids: int = 1000000000,
                time_budget_s: float = 0.0) -> dict:
        """Batched auction on (n, n) or (batch, n, n) int32 costs (numpy).
        ``scaled``: solve_auction_scaled (epsilon = epsilon0); else solve_auction."""
        c = np.ascontiguousarray(costs, dtype=np.int32)
        single = c.ndim == 2
        if single:
            c = c[None]
        b, n, n2 = c.shape
        if n != n2:
            raise ValueError("square cost matrices required")
        cfg = AuctionConfig(int(bool(scaled)), float(epsilon), float(theta), float(epsilon_final),
                            int(max_bids), float(time_budget_s))
        out = dict(prices=np.zeros((b, n)), row_to_col=np.full((b, n), -1, np.int32),
                   total_cost=np.zeros(b, np.int64), bids=np.zeros(b, np.int64),
                   converged=np.zeros(b, np.int32), epsilon_last=np.zeros(b))
        out["seconds"] = self.auction_into(c, b, n, cfg, **{k: out[k] for k in (
            "prices", "row_to_col", "total_cost", "bids", "converged", "epsilon_last")})
        if single:
            for k in ("prices", "row_to_col", "total_cost", "bids", "converged", "epsilon_last"):
                out[k] = out[k][0]
        return out

    def costs_from_points(self, a, b, scale: float, squared: bool = False, out=None):
        """The reference's build_instance (datasets.cpp:184-214) on the GPU:
        ``llround(scale * ||a_i - b_j||)`` (``squared``: the squared distance).

        ``a``: (n, dim) or (batch, n, dim), ``b`` likewise with m points; float64
        or float32 (promoted to double), numpy (host) or torch (host or cuda).
        Returns int32 costs (batch, n, m) or (n, m) in ``out`` (allocated like
        ``a`` when None).  Raises KmbError(KMB_ERANGE) when a cost overflows int32.
        """
        single = len(a.shape) == 2
        if single:
            a, b = a[None], b[None]
        if a.dtype not in (np.float64, np.float32) and str(a.dtype) not in (
                "torch.float64", "torch.float32"):
            raise ValueError("points must be float64 or float32")
        if str(a.dtype) != str(b.dtype):
            raise ValueError("a and b must share a dtype")
        if hasattr(a, "contiguous"):
            a, b = a.contiguous(), b.contiguous()
        else:
            a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
        batch, n, dim = a.shape
        if b.shape[0] != batch or b.shape[2] != dim:
            raise ValueError("point dimensions differ")
        m = b.shape[1]
        dtype = 0 if str(a.dtype).endswith("float64") else 1
        if out is None:
            if hasattr(a, "new_empty"):
                import torch
                out = torch.empty((batch, n, m), dtype=torch.int32, device=a.device)
            else:
                out = np.empty((batch, n, m), np.int32)
        self._check(self._lib.kmb_costs_from_points(
            self._h, C.c_void_p(_ptr(a)), C.c_void_p(_ptr(b)), dtype, batch, n, m, dim,
            float(scale), int(bool(squared)), C.c_void_p(_ptr(out))))
        return out[0] if single else out

    # -- numpy convenience -------------------------------------------------------
    def solve(self, cost: np.ndarray, seed: int = KMB_SEED_BATCHED,
              time_budget_s: float = 0.0) -> Result:
        """int64 input goes through kmb_solve_i64 (the reference's cost type and
        range), anything else through kmb_solve_i32."""
        wide = np.asarray(cost).dtype == np.int64
        c = np.ascontiguousarray(cost, dtype=np.int64 if wide else np.int32)
        if c.ndim != 2 or c.shape[0] != c.shape[1]:
            raise ValueError("square cost matrix required")
        n = c.shape[0]
        r2c = np.full(n, -1, np.int32)
        u = np.zeros(n, np.int64)
        v = np.zeros(n, np.int64)
        tot = np.zeros(1, np.int64)
        t0 = time.perf_counter()
        call = self.solve_i64_into if wide else self.solve_into
        st = call(c, n, n, seed, r2c, u, v, tot, time_budget_s)
        wall = time.perf_counter() - t0
        return Result(r2c, u, v, int(tot[0]), iterations=int(st.phases + st.dual_steps),
                      exact=bool(st.converged), converged=bool(st.converged), wall_seconds=wall,
                      stats=_stats_dict(st))

    def solve_batch(self, costs: np.ndarray, seed: int = KMB_SEED_BATCHED) -> Result:
        wide = np.asarray(costs).dtype == np.int64
        c = np.ascontiguousarray(costs, dtype=np.int64 if wide else np.int32)
        b, n, n2 = c.shape
        if n != n2:
            raise ValueError("square cost matrices required")
        r2c = np.full((b, n), -1, np.int32)
        u = np.zeros((b, n), np.int64)
        v = np.zeros((b, n), np.int64)
        tot = np.zeros(b, np.int64)
        t0 = time.perf_counter()
        call = self.solve_batch_i64_into if wide else self.solve_batch_into
        st = call(c, b, n, seed, r2c, u, v, tot)
        wall = time.perf_counter() - t0
        return Result(r2c, u, v, tot, iterations=int(st.phases + st.dual_steps),
                      wall_seconds=wall, stats=_stats_dict(st))


def solve_batch_multi(solvers, costs, seed: int = KMB_SEED_BATCHED) -> Result:
    """A batch split over several contexts (normally one ``Solver`` per GPU)
    through ``kmb_solve_batch_multi_i32``: contiguous equal slices, solved
    concurrently, results in batch order.  Host (numpy) buffers."""
    solvers = list(solvers)
    if not solvers:
        raise ValueError("solve_batch_multi: no solvers")
    lib = solvers[0]._lib
    c = np.ascontiguousarray(costs, dtype=np.int32)
    b, n, n2 = c.shape
    if n != n2:
        raise ValueError("square cost matrices required")
    r2c = np.full((b, n), -1, np.int32)
    u = np.zeros((b, n), np.int64)
    v = np.zeros((b, n), np.int64)
    tot = np.zeros(b, np.int64)
    hs = (C.c_void_p * len(solvers))(*[s._h for s in solvers])
    st = Stats()
    t0 = time.perf_counter()
    rc = lib.kmb_solve_batch_multi_i32(hs, len(solvers), C.c_void_p(c.ctypes.data), b, n, seed,
                                       C.c_void_p(r2c.ctypes.data), C.c_void_p(u.ctypes.data),
                                       C.c_void_p(v.ctypes.data), C.c_void_p(tot.ctypes.data),
                                       C.byref(st))
    wall = time.perf_counter() - t0
    solvers[0]._check(rc)
    return Result(r2c, u, v, tot, iterations=int(st.phases + st.dual_steps),
                  wall_seconds=wall, stats=_stats_dict(st))


def _stats_dict(st: Stats) -> dict:
    d = {k: getattr(st, k) for k, _ in Stats._fields_}
    d["stage_ns"] = list(d["stage_ns"])
    return d


_default: Solver | None = None


def default_solver() -> Solver:
    global _default
    if _default is None:
        _default = Solver(0)
    return _default


# ---- reference-shaped entry points ------------------------------------------------

def _validate(cost, supplies, demands, who: str) -> np.ndarray:
    """require_unit_square (hungarian.cpp:15-21) + validate_instance (core.cpp:30-55)
    for the assignment case, with the reference's messages."""
    c = np.asarray(cost)
    if c.ndim != 2 or c.shape[0] <= 0 or c.shape[1] <= 0:
        raise ValueError(f"{who}: dimensions must be positive")
    n, m = c.shape
    if supplies is not None and len(supplies) != n:
        raise ValueError(f"{who}: supplies size does not match n")
    if demands is not None and len(demands) != m:
        raise ValueError(f"{who}: demands size does not match m")
    if (supplies is not None and any(s <= 0 for s in supplies)):
        raise ValueError(f"{who}: supplies must be positive")
    if (demands is not None and any(d <= 0 for d in demands)):
        raise ValueError(f"{who}: demands must be positive")
    if supplies is not None and demands is not None and sum(supplies) != sum(demands):
        raise ValueError(f"{who}: total supply does not equal total demand")
    unit = n == m and (supplies is None or all(s == 1 for s in supplies)) and \
        (demands is None or all(d == 1 for d in demands))
    if not unit:
        raise ValueError(f"{who}: requires a unit-capacity square instance")
    return c


def quantize_costs(cost, B: int, solver: Solver | None = None):
    """``ot::quantize_costs`` (hungarian.cpp:33-53) on the device
    (``kmb_quantize_i64``): returns (chat = floor(C*B/N), N, lossless)."""
    if B <= 0:
        raise ValueError("quantize_costs: B must be positive")
    c = np.ascontiguousarray(cost, dtype=np.int64)
    chat = np.empty_like(c)
    try:
        N, lossless = (solver or default_solver()).quantize(c, int(B), chat)
    except KmbError as e:
        raise ValueError(str(e)) from None
    return chat, N, lossless


def solve_km(cost, supplies=None, demands=None, time_budget_s: float = 0.0,
             solver: Solver | None = None) -> Result:
    """Exact KM from u = v = 0; duals identical to ``ot::solve_km``.  int64
    costs over the reference's whole admissible range (kmb_solve_i64)."""
    c = _validate(cost, supplies, demands, "solve_km")
    s = solver or default_solver()
    try:
        r = s.solve(np.asarray(c, dtype=np.int64), KMB_SEED_KM, time_budget_s)
    except KmbError as e:
        if e.code > 0:
            raise ValueError("solve_km: " + str(e).split(": ", 1)[-1]) from None
        raise
    r.iterations = c.shape[0]  # hungarian.cpp:130: iterations = n
    return r


def solve_batched_km(cost, B: int | None = 100, supplies=None, demands=None,
                     time_budget_s: float = 0.0, solver: Solver | None = None,
                     return_quantized: bool = False):
    """``ot::solve_batched_km`` end to end on the device
    (``kmb_solve_batched_km_i64``: validation, quantization to chat, search).
    The default B = 100 is ``BatchedKMConfig{}``'s (hungarian.hpp:42-45), so a
    caller relying on the default gets the reference's (possibly lossy) answer;
    ``B=None`` (an extension) is the lossless B = N.  u, v are the duals of
    chat; ``exact`` = lossless and converged (hungarian.cpp:374-376); the total
    cost and objective are reported against the true costs."""
    c = _validate(cost, supplies, demands, "solve_batched_km")
    c64 = np.ascontiguousarray(c, dtype=np.int64)
    if B is None:
        B = max(int(c64.max()), 1)
    n = c64.shape[0]
    s = solver or default_solver()
    r2c = np.full(n, -1, np.int32)
    u = np.zeros(n, np.int64)
    v = np.zeros(n, np.int64)
    tot = np.zeros(1, np.int64)
    chat = np.empty_like(c64) if return_quantized else None
    t0 = time.perf_counter()
    try:
        st, N, lossless = s.solve_batched_km_into(c64, n, int(B), r2c, u, v, tot, chat, time_budget_s)
    except KmbError as e:
        if e.code > 0:
            raise ValueError(str(e)) from None
        raise
    wall = time.perf_counter() - t0
    r = Result(r2c, u, v, int(tot[0]), iterations=int(st.phases + st.dual_steps),
               exact=bool(lossless and st.converged), converged=bool(st.converged),
               wall_seconds=wall, stats=_stats_dict(st))
    if return_quantized:
        return r, (chat, int(B), N, lossless)
    return r


def calibrate_batch_level(cost, exact: float, target_ratio: float = 1.1,
                          solver: Solver | None = None) -> int:
    """Smallest power-of-two quantization level B whose batched-KM objective is
    within ``target_ratio`` of ``exact``; capped at the lossless B = N*n
    (the reference's calibrate_batch_level, bench.cpp:296-308).  This is the
    paper's lossy 1.1-approximate mode (Table 3)."""
    c = np.asarray(cost, dtype=np.int64)
    cap = max(int(c.max()) if c.size else 0, 1) * c.shape[0]
    B = 1
    while True:
        if B >= cap:
            return cap
        r = solve_batched_km(c, B, solver=solver)
        if r.objective <= target_ratio * exact * (1 + 1e-12):
            return B
        B *= 2


def _auction_result(c, o, n: int) -> Result:
    ok = o["row_to_col"] >= 0
    rows = np.arange(n)
    tot = int(np.asarray(c, np.int64)[rows[ok], o["row_to_col"][ok]].sum())
    conv = bool(o["converged"])
    return Result(o["row_to_col"], None, None, tot, iterations=int(o["bids"]),
                  exact=conv and float(o["epsilon_last"]) * n < 1.0, converged=conv,
                  wall_seconds=o["seconds"], prices=o["prices"])


def _auction_costs(cost, supplies, demands, who: str) -> np.ndarray:
    c = _validate(cost, supplies, demands, who)
    if (np.asarray(c) < 0).any():
        raise ValueError(f"{who}: costs must be nonnegative")
    if np.asarray(c).max() > 2**31 - 1:
        raise ValueError(f"{who}: cost exceeds the device range [0, 2^31)")
    return np.asarray(c).astype(np.int32)


def solve_auction(cost, epsilon: float = 1.0, max_bids: int = 1000000000,
                  time_budget_s: float = 0.0, supplies=None, demands=None,
                  solver: Solver | None = None) -> Result:
    """``ot::solve_auction`` (auction.cpp:186-199) on the GPU: the same bids, the
    same double prices (``Result.prices``), the same assignment; ``iterations``
    counts bids, ``exact`` = converged and n * epsilon < 1."""
    c = _auction_costs(cost, supplies, demands, "solve_auction")
    if not epsilon > 0.0:
        raise ValueError("solve_auction: epsilon must be positive")
    o = (solver or default_solver()).auction(c, False, epsilon, 4.0, 0.0, max_bids, time_budget_s)
    return _auction_result(c, o, c.shape[0])


def solve_auction_scaled(cost, epsilon0: float = 0.0, theta: float = 4.0,
                         epsilon_final: float = 0.0, max_bids: int = 1000000000,
                         time_budget_s: float = 0.0, supplies=None, demands=None,
                         solver: Solver | None = None) -> Result:
    """``ot::solve_auction_scaled`` (auction.cpp:201-229) on the GPU: epsilon
    scaling with prices carried across rounds; defaults as the reference's
    (epsilon0 <= 0: max_cost / 2; epsilon_final <= 0: 1 / (n + 1), exact)."""
    c = _auction_costs(cost, supplies, demands, "solve_auction_scaled")
    if not theta > 1.0:
        raise ValueError("solve_auction_scaled: theta must exceed 1")
    o = (solver or default_solver()).auction(c, True, epsilon0, theta, epsilon_final, max_bids,
                                             time_budget_s)
    return _auction_result(c, o, c.shape[0])


def calibrate_auction_eps(cost, exact_int: int, solver: Solver | None = None) -> float:
    """Largest epsilon_final on the doubling grid from 1/(n+1) for which the scaled
    auction still returns the exact objective (bench.cpp:310-326)."""
    c = np.asarray(cost, dtype=np.int64)
    N = float(max(int(c.max()) if c.size else 0, 1))
    eps = 1.0 / (c.shape[0] + 1)
    best = 0.0
    while eps <= N:
        r = solve_auction_scaled(c, epsilon_final=eps, solver=solver)
        if not r.converged or round(r.objective) != exact_int:
            break
        best = eps
        eps *= 2.0
    if best == 0.0:
        raise RuntimeError("auction calibration failed at epsilon = 1/(n+1)")
    return best

