"""GPU: the 64-bit cost path — the reference's own cost type (OTInstance::cost
is int64) over its whole admissible range — and the K11 quantization kernel.

* kmb_solve_i64 / kmb_solve_batch_i64: costs up to validate_instance's headroom
  (core.cpp:47-53) run on the wide engine (stats engine 9); u, v and the total
  cost are compared bit-exact with the unmodified reference (oracle/_ref), the
  assignment where the optimum is unique, exact complementary slackness always.
* kmb_quantize_i64 (quantize_costs, hungarian.cpp:33-53) against the
  reference's known answers (test_hungarian.cpp:27-59) and random vectors.
* kmb_solve_batched_km_i64: the reference's solve_batched_km end to end on the
  device, including chat values beyond the 32-bit engines' range.
"""
import numpy as np
import pytest

import oracle as O
from paper_2005_01182_b200 import KMB_SEED_BATCHED, KMB_SEED_KM, KmbError
from paper_2005_01182_b200 import api

from .test_gpu_parity import certificate_ok, optimum_unique

pytestmark = pytest.mark.gpu


def headroom(n: int) -> int:
    return ((1 << 62) // n) // (2 * n + 2)


def ref_batched(c):
    """The reference's solve_batched_km at its lossless B = N where N * N fits
    int64 (quantize_costs rejects B * N beyond it); above that, the C
    restatement of the same algorithm on C (oracle/km_oracle.c, pinned to the
    reference bit for bit in tests/test_oracle.py)."""
    hi = max(int(np.max(c)), 1)
    return O.ref_solve_batched_km(c) if hi * hi <= 2**63 - 1 else O.kmo_solve_batched(c)


def check(r, ref, c):
    assert r.total_cost == ref.total_cost
    np.testing.assert_array_equal(r.u, ref.u)
    np.testing.assert_array_equal(r.v, ref.v)
    assert certificate_ok(c, r.u, r.v, r.row_to_col)
    if optimum_unique(c, r.u, r.v, r.row_to_col):
        np.testing.assert_array_equal(r.row_to_col, ref.row_to_col)


def wide_instance(rng, n, hi):
    # a mix of huge and tiny entries so reduced costs span the whole int64 range
    c = rng.integers(0, hi, size=(n, n), dtype=np.int64)
    c[rng.random((n, n)) < 0.2] = rng.integers(0, 1000)
    return c


@pytest.mark.parametrize("seed", [KMB_SEED_KM, KMB_SEED_BATCHED])
def test_wide_engine_matches_reference(solver, seed):
    rng = np.random.default_rng(71 + seed)
    for t in range(40):
        n = int(rng.integers(1, 90))
        hi = int(rng.choice([2**29, 2**33, 2**40, headroom(n)]))
        hi = min(hi, headroom(n))
        c = wide_instance(rng, n, hi)
        c[0, 0] = hi  # pin the maximum so the wide engine runs
        ref = O.ref_solve_km(c) if seed == KMB_SEED_KM else ref_batched(c)
        r = solver.solve(c, seed)
        assert r.stats["engine"] == 9
        check(r, ref, c)


def test_wide_engine_larger_n(solver):
    rng = np.random.default_rng(5)
    for n in (255, 513, 1000):
        c = wide_instance(rng, n, headroom(n))
        ref = ref_batched(c)
        r = solver.solve(c, KMB_SEED_BATCHED)
        assert r.stats["engine"] == 9
        check(r, ref, c)


def test_i64_small_costs_run_the_32bit_engines(solver):
    rng = np.random.default_rng(9)
    for n in (3, 100, 300, 1500):
        c = rng.integers(0, 2**29, size=(n, n), dtype=np.int64)
        c[0, 0] = 2**29 - 1
        ref = O.ref_solve_batched_km(c)
        r = solver.solve(c, KMB_SEED_BATCHED)
        assert r.stats["engine"] != 9
        check(r, ref, c)


def test_i64_headroom_boundary_and_errors(solver):
    n = 7
    c = np.full((n, n), 3, np.int64)
    c[1, 2] = headroom(n)  # the largest admissible cost
    check(solver.solve(c, KMB_SEED_KM), O.ref_solve_km(c), c)
    c[1, 2] = headroom(n) + 1  # validate_instance rejects it
    with pytest.raises(O.RefError, match="supply \\* cost magnitude too large"):
        O.ref_solve_km(c)
    with pytest.raises(KmbError, match="supply \\* cost magnitude too large for 64-bit arithmetic"):
        solver.solve(c, KMB_SEED_KM)
    c[1, 2] = -5
    with pytest.raises(KmbError, match="costs must be nonnegative"):
        solver.solve(c, KMB_SEED_KM)
    with pytest.raises(ValueError, match="solve_km: costs must be nonnegative"):
        api.solve_km(c)


def test_i64_batch_mixed(solver):
    """A batch whose maximum is wide runs every instance on the wide engine;
    per-instance duals equal the reference's."""
    rng = np.random.default_rng(13)
    b, n = 37, 40
    c = rng.integers(0, 5000, size=(b, n, n), dtype=np.int64)
    c[3] = wide_instance(rng, n, headroom(n))
    c[20, 5, 5] = 2**45
    r = solver.solve_batch(c, KMB_SEED_BATCHED)
    for k in range(b):
        ref = ref_batched(c[k])
        assert r.total_cost[k] == ref.total_cost
        np.testing.assert_array_equal(r.u[k], ref.u)
        np.testing.assert_array_equal(r.v[k], ref.v)


def test_i64_time_budget_partial(solver):
    """Budget expiry on the wide engine: converged = 0, feasible duals, partial
    matching (free rows -1), like the reference's budgeted solve."""
    rng = np.random.default_rng(3)
    n = 600
    c = wide_instance(rng, n, headroom(n))
    r = solver.solve(c, KMB_SEED_BATCHED, time_budget_s=1e-9)
    assert not r.converged
    assert (r.row_to_col == -1).any()
    cc = c.astype(np.int64)
    assert ((cc - r.u[:, None] - r.v[None, :]) >= 0).all()
    m = r.row_to_col >= 0
    rows = np.nonzero(m)[0]
    assert (cc[rows, r.row_to_col[m]] == r.u[rows] + r.v[r.row_to_col[m]]).all()


# ---- K11: quantize_costs on the device ----------------------------------------

def test_quantize_known_answers(solver):  # test_hungarian.cpp:27-59
    for cost, B, chat, N, lossless in (
            ([0, 5, 10], 2, [0, 1, 2], 10, True),
            ([0, 3, 7], 10, [0, 4, 10], 7, False),
            ([0, 0, 0], 5, [0, 0, 0], 1, True),
            ([4, 8], 8, [4, 8], 8, True)):
        got, n_, ll = api.quantize_costs(np.array(cost), B, solver=solver)
        ref = O.ref_quantize_costs(cost, B)
        assert got.tolist() == list(ref[0]) and n_ == ref[1] and ll == ref[2]
        assert got.tolist() == chat and n_ == N and ll == lossless


def test_quantize_matches_reference(solver):
    rng = np.random.default_rng(1)
    for B in (1, 2, 7, 64, 999, 10**6, 2**40):
        for hi in (10**5, 2**33):
            c = rng.integers(0, hi, size=int(rng.integers(1, 5000)))
            if B > (2**63 - 1) // int(c.max()):
                continue
            a = api.quantize_costs(c, B, solver=solver)
            b = O.ref_quantize_costs(c, B)
            assert np.array_equal(a[0], b[0]) and a[1] == b[1] and a[2] == b[2]
    with pytest.raises(ValueError, match="quantize_costs: B must be positive"):
        api.quantize_costs([1], 0, solver=solver)
    with pytest.raises(ValueError, match="quantize_costs: B \\* max cost overflows"):
        api.quantize_costs([2**40], 2**40, solver=solver)


def test_batched_km_i64_wide_chat(solver):
    """solve_batched_km with B beyond the 32-bit range and not a multiple of N:
    chat itself is wide and runs on the wide engine; duals of chat, chat and the
    lossless flag equal the reference's."""
    rng = np.random.default_rng(29)
    for t in range(12):
        n = int(rng.integers(2, 60))
        c = rng.integers(0, 10**6, size=(n, n), dtype=np.int64)
        N = int(c.max())
        B = int(rng.choice([2**31 + 7, 3 * 10**9 + 1, N * n * 1000 + 1]))
        ref = O.ref_solve_batched_km(c, B=B, want_chat=True)
        r, (chat, _, N2, lossless) = api.solve_batched_km(c, B, solver=solver, return_quantized=True)
        assert r.stats["engine"] == 9
        np.testing.assert_array_equal(chat.ravel(), np.ravel(ref.chat))
        assert N2 == N and lossless == ref.exact
        np.testing.assert_array_equal(r.u, ref.u)
        np.testing.assert_array_equal(r.v, ref.v)
        assert r.total_cost == ref.total_cost or not lossless
        rows = np.arange(n)
        rc = np.reshape(ref.chat, (n, n))
        assert chat[rows, r.row_to_col].sum() == rc[rows, ref.row_to_col].sum()


def test_batched_km_i64_lossless_scaling_of_wide_costs(solver):
    """B = N * n with wide costs (test_hungarian.cpp:144-156 lifted beyond 2^29):
    the reference's exact answer, solved on C and scaled by n on the device."""
    rng = np.random.default_rng(31)
    for n in (3, 7):
        c = wide_instance(rng, n, 2**30)
        c[0, 1] = 2**30  # N = 2^30: chat = n * C exceeds 2^29 and N * B stays in int64
        N = int(c.max())
        ref = O.ref_solve_batched_km(c, B=N * n)
        r = api.solve_batched_km(c, N * n, solver=solver)
        assert r.exact and ref.exact
        assert r.total_cost == ref.total_cost
        np.testing.assert_array_equal(r.u, ref.u)
        np.testing.assert_array_equal(r.v, ref.v)
