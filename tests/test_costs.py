"""Cost construction — the caller before the path.

CPU: the reference's own build_instance (datasets.cpp:184-214, compiled into
oracle/_ref) pins the host generators' Euclidean mode (config 3), and an
explicit IEEE restatement pins the squared mode (configs 2 and 4).
GPU: kmb_costs_from_points must be bit-identical to both, on host and device
buffers, for square, rectangular and batched point sets.
"""
import numpy as np
import pytest

import oracle as O
from paper_2005_01182_b200 import workloads as W


def np_costs(a, b, scale, squared):
    """llround(scale * d(a_i, b_j)) with the dimensions summed in order, every
    op a rounded double op — the reference's euclidean() (datasets.cpp:16-22)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    s = np.zeros((a.shape[0], b.shape[0]))
    for d in range(a.shape[1]):
        diff = a[:, d][:, None] - b[:, d][None, :]
        s = s + diff * diff
    x = scale * (s if squared else np.sqrt(s))
    f = np.floor(x)  # llround for x >= 0: half away from zero
    return (f + (x - f >= 0.5)).astype(np.int64)


def test_reference_build_instance_pins_config3_generator():
    a, b, dim, scale, squared = W.points("c3", batch=2, first=5)
    want = W.CONFIGS["c3"].make(batch=2, first=5)
    for t in range(2):
        ref = O.ref_build_instance(a[t].astype(np.float64), b[t].astype(np.float64), scale)
        np.testing.assert_array_equal(ref, want[t])


@pytest.mark.parametrize("key", ["c2", "c4"])
def test_squared_generators_match_restatement(key):
    a, b, dim, scale, squared = W.points(key)
    assert squared
    want = W.CONFIGS[key].make()
    np.testing.assert_array_equal(np_costs(a, b, scale, True), want)


def test_reference_build_instance_random_points():
    rng = np.random.default_rng(7)
    a = rng.normal(size=(37, 5)) * 3
    b = rng.normal(size=(37, 5)) * 3
    np.testing.assert_array_equal(O.ref_build_instance(a, b, 997.5), np_costs(a, b, 997.5, False))


# ---------------------------------------------------------------- GPU ------
@pytest.mark.gpu
@pytest.mark.parametrize("key", ["c2", "c4"])
def test_gpu_costs_configs_2_4(solver, key):
    a, b, dim, scale, squared = W.points(key)
    got = solver.costs_from_points(a, b, scale, squared)
    np.testing.assert_array_equal(got, W.CONFIGS[key].make())


@pytest.mark.gpu
def test_gpu_costs_config3_batch(solver):
    a, b, dim, scale, squared = W.points("c3", batch=64, first=100)
    got = solver.costs_from_points(a, b, scale, squared)
    np.testing.assert_array_equal(got, W.CONFIGS["c3"].make(batch=64, first=100))


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,dim", [(1, 1, 1), (37, 37, 5), (33, 70, 31), (100, 3, 65)])
def test_gpu_costs_vs_reference_build_instance(solver, n, m, dim):
    rng = np.random.default_rng(n * 1000 + m + dim)
    a = rng.normal(size=(n, dim)) * 10
    b = rng.normal(size=(m, dim)) * 10
    got = solver.costs_from_points(a, b, 1234.5)
    np.testing.assert_array_equal(got, np_costs(a, b, 1234.5, False))
    if n == m:
        np.testing.assert_array_equal(got, O.ref_build_instance(a, b, 1234.5))


@pytest.mark.gpu
def test_gpu_costs_device_buffers_then_solve(solver):
    """Points already in HBM -> costs in HBM -> batched solve, no host hop;
    the duals match the reference on the same instances."""
    import torch
    a, b, dim, scale, squared = W.points("c3", batch=4, first=0)
    ta = torch.from_numpy(a).cuda()
    tb = torch.from_numpy(b).cuda()
    cost = solver.costs_from_points(ta, tb, scale, squared)
    assert cost.is_cuda and cost.dtype == torch.int32
    host = cost.cpu().numpy()
    np.testing.assert_array_equal(host, W.CONFIGS["c3"].make(batch=4, first=0))
    r2c = torch.empty((4, 128), dtype=torch.int32, device="cuda")
    u = torch.empty((4, 128), dtype=torch.int64, device="cuda")
    v = torch.empty((4, 128), dtype=torch.int64, device="cuda")
    tot = torch.empty(4, dtype=torch.int64, device="cuda")
    solver.solve_batch_into(cost, 4, 128, 1, r2c, u, v, tot)
    for t in range(4):
        ref = O.ref_solve_batched_km(host[t])
        np.testing.assert_array_equal(u[t].cpu().numpy(), ref.u)
        np.testing.assert_array_equal(v[t].cpu().numpy(), ref.v)
        assert int(tot[t]) == ref.total_cost


@pytest.mark.gpu
def test_gpu_costs_overflow_is_erange(solver):
    from paper_2005_01182_b200.api import KmbError
    a = np.zeros((4, 2))
    b = np.full((4, 2), 1e6)
    with pytest.raises(KmbError) as e:
        solver.costs_from_points(a, b, 1e6)
    assert e.value.code == 3


@pytest.mark.gpu
def test_gpu_costs_bad_args(solver):
    from paper_2005_01182_b200.api import KmbError
    a = np.zeros((4, 2))
    with pytest.raises(KmbError):
        solver.costs_from_points(a, a, 0.0)
    with pytest.raises(ValueError):
        solver.costs_from_points(a, np.zeros((4, 3)), 1.0)


def test_circle_square_points_match_reference_build_instance():
    """acceptance.cpp criterion 1's CircleSquare clouds through the reference's
    own build_instance reproduce the restated cost matrix."""
    from tests.golden.make_golden import circle_square, circle_square_points
    sq, ci = circle_square_points(100)
    np.testing.assert_array_equal(O.ref_build_instance(sq, ci, 1e4), circle_square(100))


@pytest.mark.gpu
@pytest.mark.parametrize("k,objective", [(100, 732033), (900, 9515106)])
def test_gpu_circle_square_acceptance(solver, k, objective):
    """acceptance.cpp criterion 1: cs100 = 732033, cs900 = 9515106,
    from the point clouds: GPU build_instance -> GPU solve (both seeds), duals
    equal to the reference's."""
    from paper_2005_01182_b200 import solve_batched_km, solve_km
    from tests.golden.make_golden import circle_square, circle_square_points
    sq, ci = circle_square_points(k)
    c = solver.costs_from_points(sq, ci, 1e4)
    np.testing.assert_array_equal(c, circle_square(k))
    r = solve_batched_km(c, None, solver=solver)  # lossless
    assert r.total_cost == objective
    ref = O.ref_solve_batched_km(c)
    np.testing.assert_array_equal(r.u, ref.u)
    np.testing.assert_array_equal(r.v, ref.v)
    rk = solve_km(c, solver=solver)
    assert rk.total_cost == objective
    refk = O.ref_solve_km(c)
    np.testing.assert_array_equal(rk.u, refk.u)
    np.testing.assert_array_equal(rk.v, refk.v)
