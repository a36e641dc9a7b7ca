"""Generate the committed golden fixtures with the reference itself.

Run here (where /root/reference exists and oracle/_ref/libotref.so is built):

    python tests/golden/make_golden.py [--with-c4] [--with-c5]

* small_cases.npz — 200 random instances (n <= 40, several value ranges) with
  the reference's solve_batched_km (lossless B) outputs: total cost, u, v.
* configs.json    — for configs 1-5: FNV-1a of the seeded int32 cost buffer,
  total cost, FNV-1a of u and v, dual-step count, and who produced them
  (c1, c2, c3[0:64], c4 by the unmodified reference; c5 by the seeded e-maxx
  restatement, which tests/test_oracle.py pins against the reference on
  configs 1-4).

Also home of the RNG-free CircleSquare restatement (datasets.cpp:57-112 +
build_instance :184-214) used to pin acceptance.cpp criterion 1's objectives.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def _llround(x: float) -> int:
    r = math.floor(x)
    return int(r + 1) if x - r >= 0.5 else int(r)


def circle_square_points(k: int) -> tuple[np.ndarray, np.ndarray]:
    """gen_circle_square(k)'s two point clouds (datasets.cpp:57-112): the s x s
    integer square centred at the origin and the k lattice points closest to
    the origin ordered by (radius^2, angle)."""
    s = int(round(math.sqrt(k)))
    assert s * s == k
    off = (s - 1) // 2
    square = [(float(x - off), float(y - off)) for y in range(s) for x in range(s)]
    R = s + 2
    cands = []
    for y in range(-R, R + 1):
        for x in range(-R, R + 1):
            r2 = x * x + y * y
            if r2 <= R * R:
                if x == 0 and y == 0:
                    a = 0.0
                else:
                    a = math.atan2(float(y), float(x))
                    if a < 0.0:
                        a += 2.0 * 3.14159265358979323846
                cands.append((r2, a, x, y))
    cands.sort()
    circle = [(float(c[2]), float(c[3])) for c in cands[:k]]
    return np.array(square, np.float64), np.array(circle, np.float64)


def circle_square(k: int, scale: float = 1e4) -> np.ndarray:
    """gen_circle_square(k) cost matrix (datasets.cpp:57-112, :184-214)."""
    square, circle = circle_square_points(k)
    c = np.empty((k, k), np.int64)
    for i, (px, py) in enumerate(square):
        for j, (qx, qy) in enumerate(circle):
            dx, dy = px - qx, py - qy
            c[i, j] = _llround(scale * math.sqrt(dx * dx + dy * dy))
    return c


def main():
    import oracle as O
    from paper_2005_01182_b200 import workloads as W

    ap = argparse.ArgumentParser()
    ap.add_argument("--with-c4", action="store_true", help="reference on c4 (~70 s)")
    ap.add_argument("--with-c5", action="store_true", help="seeded e-maxx on c5 (minutes)")
    args = ap.parse_args()

    rng = np.random.default_rng(2026)
    cnt, nmax = 200, 40
    cost = np.zeros((cnt, nmax, nmax), np.int64)
    u = np.zeros((cnt, nmax), np.int64)
    v = np.zeros((cnt, nmax), np.int64)
    tot = np.zeros(cnt, np.int64)
    ns = np.zeros(cnt, np.int32)
    for t in range(cnt):
        n = int(rng.integers(1, nmax + 1))
        hi = int(rng.choice([1, 3, 20, 1000, 10**6]))
        c = rng.integers(0, hi + 1, size=(n, n))
        r = O.ref_solve_batched_km(c)
        cost[t, :n, :n] = c
        u[t, :n] = r.u
        v[t, :n] = r.v
        tot[t] = r.total_cost
        ns[t] = n
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), count=cnt, n=ns, cost=cost, u=u,
                        v=v, total=tot)

    path = os.path.join(HERE, "configs.json")
    out = {}
    if os.path.exists(path):
        with open(path) as f:
            out = json.load(f)

    def record(key, c, r, producer, dual_steps, seconds):
        out[key] = {"cost_fnv": W.fnv1a64(c), "total_cost": int(r.total_cost),
                    "u_fnv": W.fnv1a64(np.ascontiguousarray(r.u, np.int64)),
                    "v_fnv": W.fnv1a64(np.ascontiguousarray(r.v, np.int64)),
                    "dual_steps": dual_steps, "producer": producer, "cpu_seconds": seconds}

    for key in ("c1", "c2"):
        c = W.CONFIGS[key].make()
        t0 = time.time()
        r = O.ref_solve_batched_km(c)
        dt = time.time() - t0
        ds = O.kmo_solve_batched(c).dual_steps
        record(key, c, r, "reference solve_batched_km (oracle/_ref)", ds, dt)
    c3 = W.CONFIGS["c3"].make(batch=64)
    tots, uh, vh = [], [], []
    for t in range(64):
        r = O.ref_solve_batched_km(c3[t])
        tots.append(int(r.total_cost))
        uh.append(W.fnv1a64(r.u))
        vh.append(W.fnv1a64(r.v))
    out["c3_first64"] = {"cost_fnv": W.fnv1a64(c3), "total_cost": tots, "u_fnv": uh, "v_fnv": vh,
                         "producer": "reference solve_batched_km (oracle/_ref)"}
    # every config-3 instance, by the reference on all host threads: one FNV-1a
    # over the 4096 totals, one over all u rows, one over all v rows
    c3 = W.CONFIGS["c3"].make()
    t0 = time.time()
    tot3, u3, v3, _ = O.ref_solve_many_i32(c3, mode=1, nthreads=os.cpu_count() or 1, duals=True)
    out["c3_all"] = {"cost_fnv": W.fnv1a64(c3), "total_fnv": W.fnv1a64(tot3), "u_fnv": W.fnv1a64(u3),
                     "v_fnv": W.fnv1a64(v3), "total_sum": int(tot3.sum()),
                     "producer": "reference solve_batched_km (oracle/_ref), lossless B, "
                                 f"{os.cpu_count()} threads", "cpu_seconds": time.time() - t0}
    if args.with_c4:
        c = W.CONFIGS["c4"].make()
        t0 = time.time()
        r = O.ref_solve_batched_km(c)
        dt = time.time() - t0
        record("c4", c, r, "reference solve_batched_km (oracle/_ref)", None, dt)
    if args.with_c5:
        c = W.CONFIGS["c5"].make()
        t0 = time.time()
        r = O.kmo_solve_km_seeded(c)
        dt = time.time() - t0
        record("c5", c, r, "seeded e-maxx restatement (oracle/km_oracle.c)", None, dt)
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(json.dumps({k: {kk: vv for kk, vv in v.items() if kk != "total_cost" or k != "c3_first64"}
                      for k, v in out.items() if k not in ("c3_first64",)}, indent=1))


if __name__ == "__main__":
    main()
