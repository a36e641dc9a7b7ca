"""GPU: the warp engine's 16-bit resident copy (KMB_OPT_RESIDENT16).

The validation pass of `k_warp_batch` writes every row as 16-bit offsets from
its minimum into a workspace and the search relaxes from that copy; rows whose
range does not fit 16 bits are relaxed from the int32 matrix, and an instance
with many such rows drops the copy altogether.  Whatever the mode, u, v and the
total cost must equal the unmodified reference's (hungarian.cpp:313-381,
:55-136) bit for bit, and the assignment must equal the int32 mode's (same
keys, same tie-breaking).
"""
import numpy as np
import pytest

import oracle as O
from paper_2005_01182_b200 import KMB_SEED_BATCHED, KMB_SEED_KM, KmbError
from paper_2005_01182_b200 import workloads as W
from paper_2005_01182_b200.api import OPT_ENGINE, OPT_RESIDENT16

pytestmark = pytest.mark.gpu


@pytest.fixture()
def warp16(solver):
    solver.set_option(OPT_ENGINE, 4)
    solver.set_option(OPT_RESIDENT16, 1)
    yield solver
    solver.set_option(OPT_RESIDENT16, 0)
    solver.set_option(OPT_ENGINE, 0)


def check_batch(s, c, seed):
    r = s.solve_batch(c, seed)
    assert r.stats["engine"] == 4
    for t in range(c.shape[0]):
        ref = O.ref_solve_batched_km(c[t]) if seed == KMB_SEED_BATCHED else O.ref_solve_km(c[t])
        assert r.total_cost[t] == ref.total_cost, t
        np.testing.assert_array_equal(r.u[t], ref.u)
        np.testing.assert_array_equal(r.v[t], ref.v)
    return r


@pytest.mark.parametrize("seed", [KMB_SEED_BATCHED, KMB_SEED_KM])
@pytest.mark.parametrize("n", [65, 100, 128, 129, 200, 256])
def test_resident16_matches_reference(warp16, n, seed):
    """Value ranges on both sides of 16 bits (all rows packed; some; none, which
    drops the copy per instance) and past the narrow-key range (wide keys)."""
    rng = np.random.default_rng(1000 * n + seed)
    for hi in (1000, 60000, 70000, 300000, (1 << 21) - 1, 1 << 22):
        c = rng.integers(0, hi + 1, size=(5, n, n), dtype=np.int32)
        check_batch(warp16, c, seed)


@pytest.mark.parametrize("seed", [KMB_SEED_BATCHED, KMB_SEED_KM])
def test_resident16_mixed_rows(warp16, seed):
    """A few rows per instance beyond 16 bits: they are relaxed from the int32
    matrix inside batches of packed rows."""
    rng = np.random.default_rng(7 + seed)
    c = rng.integers(0, 50000, size=(8, 128, 128), dtype=np.int32)
    for t in range(8):
        rows = rng.choice(128, size=1 + t % 7, replace=False)
        cols = rng.choice(128, size=9, replace=False)
        c[t][np.ix_(rows, cols)] += 900000
    check_batch(warp16, c, seed)
    c = rng.integers(0, 30000, size=(6, 200, 200), dtype=np.int32)
    c[:, 5, 7] = 2000000
    c[:, 199, 0] = 1500000
    check_batch(warp16, c, seed)


def test_resident16_same_assignment_as_int32(solver):
    """Config-3 instances: both modes give the same matching, duals and totals."""
    c = W.CONFIGS["c3"].make(batch=96)
    solver.set_option(OPT_ENGINE, 4)
    try:
        out = {}
        for mode in (-1, 1):
            solver.set_option(OPT_RESIDENT16, mode)
            out[mode] = solver.solve_batch(c, KMB_SEED_BATCHED)
    finally:
        solver.set_option(OPT_RESIDENT16, 0)
        solver.set_option(OPT_ENGINE, 0)
    for f in ("row_to_col", "u", "v", "total_cost"):
        np.testing.assert_array_equal(getattr(out[-1], f), getattr(out[1], f))
    assert out[-1].stats["rounds"] == out[1].stats["rounds"]
    for t in range(0, 96, 5):
        ref = O.ref_solve_batched_km(c[t])
        assert out[1].total_cost[t] == ref.total_cost
        np.testing.assert_array_equal(out[1].u[t], ref.u)


def test_resident16_host_pipeline(solver):
    """A host batch of >= 256 instances is solved in chunks as its copy lands;
    each chunk packs into its own slice of the workspace."""
    c = W.CONFIGS["c3"].make(batch=320)
    solver.set_option(OPT_ENGINE, 4)
    try:
        out = {}
        for mode in (-1, 1):
            solver.set_option(OPT_RESIDENT16, mode)
            out[mode] = solver.solve_batch(c, KMB_SEED_BATCHED)
    finally:
        solver.set_option(OPT_RESIDENT16, 0)
        solver.set_option(OPT_ENGINE, 0)
    for f in ("row_to_col", "u", "v", "total_cost"):
        np.testing.assert_array_equal(getattr(out[-1], f), getattr(out[1], f))
    for t in (0, 63, 64, 159, 160, 255, 256, 319):
        ref = O.ref_solve_batched_km(c[t])
        assert out[1].total_cost[t] == ref.total_cost
        np.testing.assert_array_equal(out[1].u[t], ref.u)
        np.testing.assert_array_equal(out[1].v[t], ref.v)


def test_resident16_large_batch_8_columns_a_lane(solver):
    """n > 128 with more instances than 16 warps per SM hold: the 72-register
    build of the 8-columns-a-lane kernel (smaller batches run the 128-register
    one), both row modes."""
    rng = np.random.default_rng(11)
    c = rng.integers(0, 3001, size=(2400, 136, 136), dtype=np.int32)
    solver.set_option(OPT_ENGINE, 4)
    try:
        out = {}
        for mode in (-1, 1):
            solver.set_option(OPT_RESIDENT16, mode)
            out[mode] = solver.solve_batch(c, KMB_SEED_BATCHED)
    finally:
        solver.set_option(OPT_RESIDENT16, 0)
        solver.set_option(OPT_ENGINE, 0)
    for f in ("row_to_col", "u", "v", "total_cost"):
        np.testing.assert_array_equal(getattr(out[-1], f), getattr(out[1], f))
    for t in range(0, 2400, 97):
        ref = O.ref_solve_batched_km(c[t])
        assert out[1].total_cost[t] == ref.total_cost
        np.testing.assert_array_equal(out[1].u[t], ref.u)
        np.testing.assert_array_equal(out[1].v[t], ref.v)


def test_resident16_invalid_instances(warp16):
    """Negative and out-of-range entries are reported per instance; the others
    of the batch are solved."""
    rng = np.random.default_rng(3)
    c = rng.integers(0, 40000, size=(6, 128, 128), dtype=np.int32)
    c[1, 3, 4] = -5
    c[4, 100, 2] = 1 << 29
    with pytest.raises(KmbError):
        warp16.solve_batch(c, KMB_SEED_BATCHED)
    good = np.ascontiguousarray(c[[0, 2, 3, 5]])
    check_batch(warp16, good, KMB_SEED_BATCHED)


def test_resident16_option_range(solver):
    with pytest.raises(KmbError):
        solver.set_option(OPT_RESIDENT16, 2)
    solver.set_option(OPT_RESIDENT16, 0)
