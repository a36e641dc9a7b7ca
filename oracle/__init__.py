"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU checkers.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_2005_01182_b200``) never does: its solve path is the CUDA
library and fails loudly when that library is missing.

Three checkers live here:

* ``ref_*``      — the UNMODIFIED reference (``/root/reference/proj/src/
  {core,hungarian}.cpp``) compiled by ``oracle/Makefile`` into
  ``oracle/_ref/libotref.so`` (``oracle/ref_capi.cpp`` is the C shim).
* ``kmo_*``      — ``km_oracle.c``: a plain-C restatement of hungarian.cpp
  (``solve_km`` :55-136, ``solve_batched_km`` :313-381, ``quantize_costs``
  :33-53) with dual-step instrumentation, plus a seeded e-maxx KM for n=16384.
* ``mirror_*``   — ``kmb_mirror.c``: the GPU engine restated step by step on
  the CPU (debugging aid, not the oracle).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libotref.so")
ORACLE_SO = os.path.join(HERE, "libkmoracle.so")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def build(quiet: bool = True) -> None:
    """Build the checkers (``make -C oracle``).  Without /root/reference the
    prebuilt ``_ref/libotref.so`` is kept as is."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


_ref = None
_orc = None


def _load_ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle` where /root/reference exists")
        lib = C.CDLL(REF_SO)
        lib.otref_last_error.restype = C.c_char_p
        lib.otref_solve_km.argtypes = [
            _i64p, C.c_int32, C.c_void_p, C.c_void_p, C.c_double, _i64p, _i64p, _i32p,
            C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_int64), _i32p,
            C.POINTER(C.c_double)]
        lib.otref_solve_batched_km.argtypes = [
            _i64p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_double, _i64p, _i64p,
            C.c_void_p, _i32p, C.POINTER(C.c_int64), C.POINTER(C.c_double),
            C.POINTER(C.c_int64), _i32p, C.POINTER(C.c_double)]
        lib.otref_quantize_costs.argtypes = [
            _i64p, C.c_int64, C.c_int64, _i64p, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        _f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
        lib.otref_build_instance.argtypes = [_f64p, C.c_int32, _f64p, C.c_int32, C.c_int32,
                                             C.c_double, _i64p]
        lib.otref_solve_auction.argtypes = [
            _i64p, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_int64,
            C.c_double, _f64p, _i32p, C.POINTER(C.c_int64), C.POINTER(C.c_double),
            C.POINTER(C.c_int64), _i32p, C.POINTER(C.c_double)]
        lib.otref_solve_many_i32.argtypes = [
            _i32p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _i64p, C.c_void_p, C.c_void_p,
            C.POINTER(C.c_double)]
        _ref = lib
    return _ref


def _load_oracle():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        lib.kmo_quantize.argtypes = [_i64p, C.c_int64, C.c_int64, _i64p,
                                     C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        lib.kmo_solve_km.argtypes = [_i64p, C.c_int32, _i64p, _i64p, _i32p, C.POINTER(C.c_int64)]
        lib.kmo_solve_batched.argtypes = [
            _i64p, C.c_int32, _i64p, _i64p, _i32p, C.POINTER(C.c_int64),
            C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_void_p, C.c_int64]
        lib.kmo_solve_km_seeded.argtypes = [_i32p, C.c_int32, _i64p, _i64p, _i32p,
                                            C.POINTER(C.c_int64)]
        lib.kmm_solve.argtypes = [
            _i32p, C.c_int32, C.c_int32, C.c_int32, _i64p, _i64p, _i32p,
            C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
            C.POINTER(C.c_int64), C.c_void_p, C.c_int64]
        lib.kmm_solve_incr.argtypes = [
            _i32p, C.c_int32, C.c_int32, _i64p, _i64p, _i32p, C.POINTER(C.c_int64),
            C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
            C.POINTER(C.c_int64), C.c_void_p, C.c_int64]
        lib.kmo_auction.argtypes = [
            _i64p, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_int64,
            np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS"), _i32p,
            C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        _orc = lib
    return _orc


class RefError(Exception):
    """Raised with the reference's own exception message."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code  # 1 invalid_argument, 2 logic_error, 3 other


@dataclass
class Solution:
    row_to_col: np.ndarray
    u: np.ndarray
    v: np.ndarray
    total_cost: int
    objective: float = 0.0
    iterations: int = 0
    exact: bool = True
    converged: bool = True
    wall_seconds: float = 0.0
    phases: int = 0
    dual_steps: int = 0
    rows_scanned: int = 0
    trace: np.ndarray | None = field(default=None, repr=False)
    chat: np.ndarray | None = field(default=None, repr=False)
    prices: np.ndarray | None = field(default=None, repr=False)


def _sq(cost) -> tuple[np.ndarray, int]:
    c = np.ascontiguousarray(cost)
    if c.ndim != 2 or c.shape[0] != c.shape[1]:
        raise ValueError("square cost matrix required")
    return c, c.shape[0]


def ref_solve_km(cost, supplies=None, demands=None, time_budget_s: float = 0.0) -> Solution:
    """The reference ``ot::solve_km`` (hungarian.cpp:55-136), unmodified."""
    lib = _load_ref()
    c, n = _sq(np.asarray(cost, dtype=np.int64))
    u = np.zeros(n, np.int64); v = np.zeros(n, np.int64); r2c = np.full(n, -1, np.int32)
    tot = C.c_int64(); obj = C.c_double(); it = C.c_int64(); ec = np.zeros(2, np.int32)
    wall = C.c_double()
    sp = None if supplies is None else np.ascontiguousarray(supplies, np.int64)
    dp = None if demands is None else np.ascontiguousarray(demands, np.int64)
    rc = lib.otref_solve_km(c, n, None if sp is None else sp.ctypes.data,
                            None if dp is None else dp.ctypes.data, time_budget_s,
                            u, v, r2c, C.byref(tot), C.byref(obj), C.byref(it), ec, C.byref(wall))
    if rc:
        raise RefError(rc, lib.otref_last_error().decode())
    return Solution(r2c, u, v, tot.value, obj.value, it.value, bool(ec[0]), bool(ec[1]), wall.value)


def ref_solve_batched_km(cost, B: int | None = None, supplies=None, demands=None,
                         time_budget_s: float = 0.0, want_chat: bool = False) -> Solution:
    """The reference ``ot::solve_batched_km`` (hungarian.cpp:313-381), unmodified.
    ``B=None`` means the lossless B = max(N, 1) (identity quantization)."""
    lib = _load_ref()
    c, n = _sq(np.asarray(cost, dtype=np.int64))
    if B is None:
        B = max(int(c.max()) if c.size else 0, 1)
    u = np.zeros(n, np.int64); v = np.zeros(n, np.int64); r2c = np.full(n, -1, np.int32)
    chat = np.zeros(c.size, np.int64) if want_chat else None
    tot = C.c_int64(); obj = C.c_double(); it = C.c_int64(); ec = np.zeros(2, np.int32)
    wall = C.c_double()
    sp = None if supplies is None else np.ascontiguousarray(supplies, np.int64)
    dp = None if demands is None else np.ascontiguousarray(demands, np.int64)
    rc = lib.otref_solve_batched_km(c, n, None if sp is None else sp.ctypes.data,
                                    None if dp is None else dp.ctypes.data, int(B), time_budget_s,
                                    u, v, None if chat is None else chat.ctypes.data, r2c,
                                    C.byref(tot), C.byref(obj), C.byref(it), ec, C.byref(wall))
    if rc:
        raise RefError(rc, lib.otref_last_error().decode())
    s = Solution(r2c, u, v, tot.value, obj.value, it.value, bool(ec[0]), bool(ec[1]), wall.value)
    if chat is not None:
        s.chat = chat.reshape(n, n)
    return s


def ref_quantize_costs(cost, B: int):
    """The reference ``ot::quantize_costs`` (hungarian.cpp:33-53)."""
    lib = _load_ref()
    c = np.ascontiguousarray(np.asarray(cost, dtype=np.int64).ravel())
    chat = np.zeros(max(c.size, 1), np.int64)
    N = C.c_int64(); ll = C.c_int32()
    rc = lib.otref_quantize_costs(c, c.size, int(B), chat, C.byref(N), C.byref(ll))
    if rc:
        raise RefError(rc, lib.otref_last_error().decode())
    return chat[: c.size], N.value, bool(ll.value)


def ref_solve_auction(cost, epsilon: float = 1.0, max_bids: int = 1000000000,
                      time_budget_s: float = 0.0) -> Solution:
    """The reference ``ot::solve_auction`` (auction.cpp:186-199), unmodified.
    ``iterations`` = bids; ``prices`` = the final column prices."""
    return _ref_auction(cost, 0, epsilon, 0.0, 0.0, max_bids, time_budget_s)


def ref_solve_auction_scaled(cost, epsilon0: float = 0.0, theta: float = 4.0,
                             epsilon_final: float = 0.0, max_bids: int = 1000000000,
                             time_budget_s: float = 0.0) -> Solution:
    """The reference ``ot::solve_auction_scaled`` (auction.cpp:201-229), unmodified."""
    return _ref_auction(cost, 1, epsilon0, theta, epsilon_final, max_bids, time_budget_s)


def _ref_auction(cost, scaled, e0, theta, ef, max_bids, budget) -> Solution:
    lib = _load_ref()
    c, n = _sq(np.asarray(cost, dtype=np.int64))
    p = np.zeros(max(n, 1), np.float64); r2c = np.full(max(n, 1), -1, np.int32)
    tot = C.c_int64(); obj = C.c_double(); it = C.c_int64(); ec = np.zeros(2, np.int32)
    wall = C.c_double()
    rc = lib.otref_solve_auction(c, n, scaled, e0, theta, ef, int(max_bids), budget, p, r2c,
                                 C.byref(tot), C.byref(obj), C.byref(it), ec, C.byref(wall))
    if rc:
        raise RefError(rc, lib.otref_last_error().decode())
    z = np.zeros(n, np.int64)
    return Solution(r2c[:n], z, z, tot.value, obj.value, it.value, bool(ec[0]), bool(ec[1]),
                    wall.value, prices=p[:n])


def kmo_auction(cost, scaled: bool = False, epsilon: float = 1.0, theta: float = 4.0,
                epsilon_final: float = 0.0, max_bids: int = 1000000000) -> Solution:
    """The C restatement of auction.cpp (oracle/auction_oracle.c).  For
    ``scaled`` the epsilon argument is epsilon0 (<= 0: default schedule)."""
    lib = _load_oracle()
    c, n = _sq(np.asarray(cost, dtype=np.int64))
    p = np.zeros(n, np.float64); r2c = np.full(n, -1, np.int32)
    bids = C.c_int64(); comp = C.c_int32(); eps = C.c_double()
    rc = lib.kmo_auction(c, n, int(scaled), epsilon, theta, epsilon_final, int(max_bids), p, r2c,
                         C.byref(bids), C.byref(comp), C.byref(eps))
    if rc:
        raise ValueError("kmo_auction: invalid arguments")
    tot = int(sum(int(c[i, r2c[i]]) for i in range(n) if r2c[i] >= 0))
    z = np.zeros(n, np.int64)
    done = bool(comp.value)
    return Solution(r2c, z, z, tot, float(tot), bids.value, done and eps.value * n < 1.0, done,
                    prices=p)


def ref_build_instance(a, b, scale: float) -> np.ndarray:
    """The reference's build_instance (datasets.cpp:184-214) on unit-weight
    point clouds: llround(scale * Euclidean distance), int64 n x m."""
    lib = _load_ref()
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    n, dim = a.shape
    m = b.shape[0]
    out = np.zeros(n * m, np.int64)
    rc = lib.otref_build_instance(a, n, b, m, dim, float(scale), out)
    if rc:
        raise RefError(rc, lib.otref_last_error().decode())
    return out.reshape(n, m)


def ref_solve_many_i32(costs: np.ndarray, mode: int = 1, nthreads: int = 1, duals: bool = False):
    """Reference solver over a batch of int32 instances on ``nthreads`` host
    threads (mode 1 = solve_batched_km at lossless B, 0 = solve_km).
    Returns (total_costs[int64 batch], wall_seconds), or with ``duals`` also
    u and v (int64, batch x n each)."""
    lib = _load_ref()
    c = np.ascontiguousarray(costs, dtype=np.int32)
    b, n, _ = c.shape
    tot = np.zeros(b, np.int64); wall = C.c_double()
    u = np.zeros((b, n), np.int64) if duals else None
    v = np.zeros((b, n), np.int64) if duals else None
    rc = lib.otref_solve_many_i32(c, b, n, mode, nthreads, tot,
                                  None if u is None else u.ctypes.data,
                                  None if v is None else v.ctypes.data, C.byref(wall))
    if rc:
        raise RefError(rc, lib.otref_last_error().decode())
    if duals:
        return tot, u, v, wall.value
    return tot, wall.value


# ---- plain-C restatement --------------------------------------------------

def kmo_quantize(cost, B: int):
    lib = _load_oracle()
    c = np.ascontiguousarray(np.asarray(cost, dtype=np.int64).ravel())
    chat = np.zeros(max(c.size, 1), np.int64)
    N = C.c_int64(); ll = C.c_int32()
    rc = lib.kmo_quantize(c, c.size, int(B), chat, C.byref(N), C.byref(ll))
    if rc == 1:
        raise ValueError("quantize_costs: B must be positive")
    if rc == 2:
        raise ValueError("quantize_costs: B * max cost overflows")
    return chat[: c.size], N.value, bool(ll)


def kmo_solve_km(cost) -> Solution:
    lib = _load_oracle()
    c, n = _sq(np.asarray(cost, dtype=np.int64))
    u = np.zeros(n, np.int64); v = np.zeros(n, np.int64); r2c = np.full(n, -1, np.int32)
    tot = C.c_int64()
    if lib.kmo_solve_km(c, n, u, v, r2c, C.byref(tot)):
        raise RuntimeError("kmo_solve_km failed")
    return Solution(r2c, u, v, tot.value, iterations=n)


def kmo_solve_batched(chat, trace_cap: int = 0) -> Solution:
    """Restated solve_batched_km on an already-quantized matrix (B = N)."""
    lib = _load_oracle()
    c, n = _sq(np.asarray(chat, dtype=np.int64))
    u = np.zeros(n, np.int64); v = np.zeros(n, np.int64); r2c = np.full(n, -1, np.int32)
    tot = C.c_int64(); ph = C.c_int64(); ds = C.c_int64()
    tr = np.zeros(2 * max(trace_cap, 1), np.int64)
    rc = lib.kmo_solve_batched(c, n, u, v, r2c, C.byref(tot), C.byref(ph), C.byref(ds),
                               tr.ctypes.data if trace_cap else None, trace_cap)
    if rc == -3:
        raise RuntimeError("batched km: no augmenting path after search")
    if rc:
        raise RuntimeError(f"kmo_solve_batched failed ({rc})")
    s = Solution(r2c, u, v, tot.value, iterations=ph.value + ds.value, phases=ph.value,
                 dual_steps=ds.value)
    if trace_cap:
        s.trace = tr[: 2 * min(ds.value, trace_cap)].reshape(-1, 2)
    return s


def kmo_solve_km_seeded(cost) -> Solution:
    lib = _load_oracle()
    c, n = _sq(np.asarray(cost, dtype=np.int32))
    u = np.zeros(n, np.int64); v = np.zeros(n, np.int64); r2c = np.full(n, -1, np.int32)
    tot = C.c_int64()
    if lib.kmo_solve_km_seeded(c, n, u, v, r2c, C.byref(tot)):
        raise RuntimeError("kmo_solve_km_seeded failed")
    return Solution(r2c, u, v, tot.value)


def mirror_solve(cost, seed: int = 1, continue_bfs: bool = False, trace_cap: int = 0) -> Solution:
    """CPU mirror of the GPU engine (seed 1 = batched reductions, 0 = u=v=0)."""
    lib = _load_oracle()
    c, n = _sq(np.asarray(cost, dtype=np.int32))
    u = np.zeros(n, np.int64); v = np.zeros(n, np.int64); r2c = np.full(n, -1, np.int32)
    tot = C.c_int64(); ph = C.c_int64(); ds = C.c_int64(); rs = C.c_int64()
    tr = np.zeros(2 * max(trace_cap, 1), np.int64)
    rc = lib.kmm_solve(c, n, seed, int(continue_bfs), u, v, r2c, C.byref(tot), C.byref(ph),
                       C.byref(ds), C.byref(rs), tr.ctypes.data if trace_cap else None, trace_cap)
    if rc:
        raise RuntimeError(f"kmm_solve failed ({rc})")
    s = Solution(r2c, u, v, tot.value, iterations=ph.value + ds.value, phases=ph.value,
                 dual_steps=ds.value, rows_scanned=rs.value)
    if trace_cap:
        s.trace = tr[: 2 * min(ds.value, trace_cap)].reshape(-1, 2)
    return s


def mirror_solve_incr(cost, seed: int = 1, trace_cap: int = 0) -> Solution:
    """CPU mirror of the engine's incremental-epoch schedule (kmm_solve_incr)."""
    lib = _load_oracle()
    c, n = _sq(np.asarray(cost, dtype=np.int32))
    u = np.zeros(n, np.int64); v = np.zeros(n, np.int64); r2c = np.full(n, -1, np.int32)
    tot = C.c_int64(); ep = C.c_int64(); ds = C.c_int64(); rs = C.c_int64(); ro = C.c_int64()
    tr = np.zeros(2 * max(trace_cap, 1), np.int64)
    rc = lib.kmm_solve_incr(c, n, seed, u, v, r2c, C.byref(tot), C.byref(ep), C.byref(ds),
                            C.byref(rs), C.byref(ro), tr.ctypes.data if trace_cap else None,
                            trace_cap)
    if rc:
        raise RuntimeError(f"kmm_solve_incr failed ({rc})")
    s = Solution(r2c, u, v, tot.value, iterations=ep.value + ds.value, phases=ep.value,
                 dual_steps=ds.value, rows_scanned=rs.value)
    s.rounds = ro.value
    if trace_cap:
        s.trace = tr[: 2 * min(ds.value, trace_cap)].reshape(-1, 2)
    return s
