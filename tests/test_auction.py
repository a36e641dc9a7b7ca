"""Auction: ot::solve_auction / ot::solve_auction_scaled.

Bar: bit-identical to the reference compiled from its sources (oracle/_ref) —
the same bid count, the same double prices (compared as bit patterns), the
same assignment, converged/exact flags — for plain and epsilon-scaled
auctions, bid budgets, and every group size of the GPU engine (warp: n <= 256,
256 threads: n <= 4096, 1024 threads above).

CPU: the C restatement (oracle/auction_oracle.c) is pinned against the
reference, and both against the reference's own test cases (test_auction.cpp).
GPU: kmb_auction_i32 against the reference on the same inputs.
"""
import numpy as np
import pytest

import oracle as O
from paper_2005_01182_b200 import workloads as W


def same(ref, got_prices, got_r2c, got_bids, got_conv=None):
    assert int(got_bids) == ref.iterations
    np.testing.assert_array_equal(np.asarray(got_prices).view(np.int64), ref.prices.view(np.int64))
    np.testing.assert_array_equal(np.asarray(got_r2c), ref.row_to_col)
    if got_conv is not None:
        assert bool(got_conv) == ref.converged


def random_cases(seed, count, nmax=40):
    rng = np.random.default_rng(seed)
    for _ in range(count):
        n = int(rng.integers(1, nmax))
        hi = int(rng.choice([1, 3, 10, 1000, 10**6]))
        yield rng.integers(0, hi, (n, n)), float(rng.choice([0.05, 0.4, 1.0, 2.5, 10.0]))


def unit_2x2():  # test_auction.cpp:17-24
    return np.array([[1, 3], [2, 1]])


def contested(n=20):  # test_auction.cpp "prices persist" case
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    return 100 * j + (i * 7 + j * 13) % 5


# ------------------------------------------------------------------ CPU ----
def test_oracle_matches_reference_random():
    for c, eps in random_cases(11, 250):
        r = O.ref_solve_auction(c, eps)
        o = O.kmo_auction(c, False, eps)
        same(r, o.prices, o.row_to_col, o.iterations, o.converged)
        assert o.exact == r.exact
        rs = O.ref_solve_auction_scaled(c)
        os_ = O.kmo_auction(c, True, 0.0)
        same(rs, os_.prices, os_.row_to_col, os_.iterations, os_.converged)
        assert os_.exact == rs.exact


def test_oracle_matches_reference_budgets_and_schedules():
    rng = np.random.default_rng(5)
    for t in range(60):
        n = int(rng.integers(2, 30))
        c = rng.integers(0, 1000, (n, n))
        mb = int(rng.integers(1, 4 * n))
        r = O.ref_solve_auction(c, 0.1, max_bids=mb)
        o = O.kmo_auction(c, False, 0.1, max_bids=mb)
        same(r, o.prices, o.row_to_col, o.iterations, o.converged)
        e0, th, ef = float(rng.choice([0.0, 50.0, 3.0])), float(rng.choice([2.0, 4.0, 7.5])), \
            float(rng.choice([0.0, 0.5, 2.0]))
        r = O.ref_solve_auction_scaled(c, e0, th, ef, max_bids=mb * 5)
        o = O.kmo_auction(c, True, e0, th, ef, max_bids=mb * 5)
        same(r, o.prices, o.row_to_col, o.iterations, o.converged)


def test_reference_known_answers():  # test_auction.cpp
    r = O.ref_solve_auction(unit_2x2(), 0.4)
    assert r.objective == 2.0 and r.exact and r.converged
    r = O.ref_solve_auction(np.full((5, 5), 3), 1.0)
    assert r.objective == 15.0
    r = O.ref_solve_auction_scaled(unit_2x2(), 4.0, 4.0, 0.4)
    assert r.objective == 2.0
    cold = O.ref_solve_auction(contested(), 0.9 / 20)
    scaled = O.ref_solve_auction_scaled(contested())
    assert cold.objective == scaled.objective and scaled.iterations < cold.iterations
    r = O.ref_solve_auction(np.random.default_rng(59).integers(0, 1000, (40, 40)), 0.1, max_bids=5)
    assert not r.converged and not r.exact
    with pytest.raises(O.RefError):
        O.ref_solve_auction(unit_2x2(), 0.0)
    with pytest.raises(O.RefError):
        O.ref_solve_auction_scaled(unit_2x2(), theta=1.0)


def test_scaled_exact_matches_km():  # "default schedule is exact" (test_auction.cpp)
    for c, _ in random_cases(61, 20, 26):
        r = O.ref_solve_auction_scaled(c)
        assert r.converged and r.exact
        assert r.total_cost == O.ref_solve_km(c).total_cost


# ------------------------------------------------------------------ GPU ----
@pytest.mark.gpu
@pytest.mark.parametrize("scaled", [False, True])
def test_gpu_random_vs_reference(solver, scaled):
    for c, eps in random_cases(23 + scaled, 150):
        o = solver.auction(c, scaled, 0.0 if scaled else eps)
        r = O.ref_solve_auction_scaled(c) if scaled else O.ref_solve_auction(c, eps)
        same(r, o["prices"], o["row_to_col"], o["bids"], o["converged"])
        assert int(o["total_cost"]) == r.total_cost


@pytest.mark.gpu
def test_gpu_known_answers(solver):
    from paper_2005_01182_b200 import solve_auction, solve_auction_scaled
    r = solve_auction(unit_2x2(), 0.4, solver=solver)
    assert r.objective == 2.0 and r.exact and r.converged
    assert solve_auction(np.full((5, 5), 3), 1.0, solver=solver).objective == 15.0
    assert solve_auction_scaled(unit_2x2(), 4.0, 4.0, 0.4, solver=solver).objective == 2.0
    cold = solve_auction(contested(), 0.9 / 20, solver=solver)
    sc = solve_auction_scaled(contested(), solver=solver)
    assert cold.objective == sc.objective and sc.iterations < cold.iterations
    same(O.ref_solve_auction(contested(), 0.9 / 20), cold.prices, cold.row_to_col, cold.iterations)
    r = solve_auction(np.random.default_rng(59).integers(0, 1000, (40, 40)), 0.1, max_bids=5,
                      solver=solver)
    assert not r.converged and not r.exact and r.iterations == 5


@pytest.mark.gpu
def test_gpu_budgets_and_schedules(solver):
    rng = np.random.default_rng(5)
    for t in range(40):
        n = int(rng.integers(2, 30))
        c = rng.integers(0, 1000, (n, n))
        mb = int(rng.integers(1, 4 * n))
        o = solver.auction(c, False, 0.1, max_bids=mb)
        same(O.ref_solve_auction(c, 0.1, max_bids=mb), o["prices"], o["row_to_col"], o["bids"],
             o["converged"])
        e0, th, ef = float(rng.choice([0.0, 50.0, 3.0])), float(rng.choice([2.0, 4.0, 7.5])), \
            float(rng.choice([0.0, 0.5, 2.0]))
        o = solver.auction(c, True, e0, th, ef, max_bids=mb * 5)
        same(O.ref_solve_auction_scaled(c, e0, th, ef, max_bids=mb * 5), o["prices"],
             o["row_to_col"], o["bids"], o["converged"])


@pytest.mark.gpu
def test_gpu_batch_config3_subset(solver):
    c = W.CONFIGS["c3"].make(batch=32, first=7)
    o = solver.auction(c, True)
    for t in range(c.shape[0]):
        r = O.ref_solve_auction_scaled(c[t])
        same(r, o["prices"][t], o["row_to_col"][t], o["bids"][t], o["converged"][t])
        assert r.exact and int(o["total_cost"][t]) == r.total_cost


@pytest.mark.gpu
def test_gpu_config1(solver):
    c = W.CONFIGS["c1"].make()
    for scaled, eps in [(True, 0.0), (False, 1.0)]:
        o = solver.auction(c, scaled, eps)
        r = O.ref_solve_auction_scaled(c) if scaled else O.ref_solve_auction(c, eps)
        same(r, o["prices"], o["row_to_col"], o["bids"], o["converged"])


@pytest.mark.gpu
@pytest.mark.parametrize("n,hi", [(257, 1000), (1000, 10**6), (4097, 1000)])
def test_gpu_cta_groups(solver, n, hi):
    c = np.random.default_rng(n).integers(0, hi, (n, n))
    o = solver.auction(c, True)
    r = O.ref_solve_auction_scaled(c)
    same(r, o["prices"], o["row_to_col"], o["bids"], o["converged"])


@pytest.mark.gpu
def test_gpu_ragged_batch_sizes(solver):
    for n in (1, 2, 3, 31, 32, 33, 63, 65, 255, 256):
        c = np.random.default_rng(n).integers(0, 50, (3, n, n))
        o = solver.auction(c, True)
        for t in range(3):
            same(O.ref_solve_auction_scaled(c[t]), o["prices"][t], o["row_to_col"][t],
                 o["bids"][t], o["converged"][t])


@pytest.mark.gpu
def test_gpu_errors(solver):
    from paper_2005_01182_b200 import solve_auction, solve_auction_scaled
    from paper_2005_01182_b200.api import KmbError
    with pytest.raises(ValueError, match="epsilon must be positive"):
        solve_auction(unit_2x2(), 0.0, solver=solver)
    with pytest.raises(ValueError, match="theta must exceed 1"):
        solve_auction_scaled(unit_2x2(), theta=1.0, solver=solver)
    with pytest.raises(ValueError, match="nonnegative"):
        solve_auction(np.array([[1, -1], [0, 0]]), solver=solver)
    with pytest.raises(KmbError) as e:  # through the C ABI: device-side validation
        solver.auction(np.array([[[1, -1], [0, 0]]]), False, 1.0)
    assert e.value.code == 2
    with pytest.raises(ValueError, match="unit-capacity"):
        solve_auction(unit_2x2(), supplies=[2, 1], demands=[1, 2], solver=solver)


@pytest.mark.gpu
def test_gpu_calibrate_matches_reference_procedure(solver):
    from paper_2005_01182_b200 import calibrate_auction_eps
    c = W.CONFIGS["c3"].make(batch=1, first=3)[0]
    exact = O.ref_solve_km(c).total_cost

    def ref_calibrate():  # bench.cpp:310-326 over the reference solver
        N = float(max(int(c.max()), 1))
        eps, best = 1.0 / (c.shape[0] + 1), 0.0
        while eps <= N:
            r = O.ref_solve_auction_scaled(c, epsilon_final=eps)
            if not r.converged or round(r.objective) != exact:
                break
            best, eps = eps, eps * 2.0
        return best

    assert calibrate_auction_eps(c, exact, solver=solver) == ref_calibrate()


@pytest.mark.gpu
def test_gpu_time_budget_partial_result(solver):
    """auction.cpp:140-144: the clock is checked every 1024 bids and an expired
    budget returns the partial matching with converged = false.  (Where the
    clock starts differs — the reference's host clock before the run, the
    kernel's at instance start — so the stopping bid is not compared.)"""
    c = W.CONFIGS["c2"].make()
    full = O.ref_solve_auction(c, 1.0)
    o = solver.auction(c, False, 1.0, time_budget_s=1e-7)
    assert not o["converged"]
    assert int(o["bids"]) % 1024 == 0 and int(o["bids"]) < full.iterations
    r2c = o["row_to_col"][o["row_to_col"] >= 0]
    assert len(np.unique(r2c)) == len(r2c)  # a partial matching
