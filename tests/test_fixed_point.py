"""Fixed-point driver pieces: host indicator / load vector (CPU) and the full
device driver vs the reference's fixed_point_solve (GPU)."""

import numpy as np
import pytest

from cases import load

SWEEPS = ["fp_1d_off", "fp_1d_su", "fp_2d_su"]


def pulse_source(x, t):
    return 1.0 * (x[:, 0] < 0.1) * (t < 0.05)


def problem_for(g, name, D=1e-3):
    import paper_2311_17500_b200.spaces as sp
    from paper_2311_17500_b200.problem import BoxGeometry, MonodomainProblem
    d, p = int(g[name + "_d"]), int(g[name + "_p"])
    st = sp.SpaceTimeSpace([sp.SplineSpace.uniform(p, int(n)) for n in g[name + "_ne"]],
                           sp.SplineSpace.uniform(p, int(g[name + "_ne_t"])))
    return MonodomainProblem(BoxGeometry([1.0] * d, 1.0), st, source=pulse_source, D=D)


def test_compute_theta_matches_reference():
    import paper_2311_17500_b200.spaces as sp
    from paper_2311_17500_b200.problem import BoxGeometry, MonodomainProblem, host_compute_theta as compute_theta
    g = load("fixed_point")
    st = sp.SpaceTimeSpace([sp.SplineSpace.uniform(2, 5), sp.SplineSpace.uniform(3, 4)], sp.SplineSpace.uniform(2, 6))
    prob = MonodomainProblem(BoxGeometry([1.0, 1.0], 2.0), st, source=pulse_source, D=1e-2)
    th = compute_theta(prob, g["theta_u"], g["theta_w"])
    np.testing.assert_allclose(th.values, g["theta_values"], rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("name", SWEEPS)
def test_load_vector_matches_reference(name):
    from paper_2311_17500_b200.problem import load_vector
    g = load("fixed_point")
    prob = problem_for(g, name)
    f = load_vector(prob.space, prob.geometry, prob.source)
    ref = g[name + "_f"]
    assert np.linalg.norm(f - ref) / np.linalg.norm(ref) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("name", SWEEPS)
def test_fixed_point_solve_matches_reference(name):
    from paper_2311_17500_b200.fixed_point import fixed_point_solve
    from paper_2311_17500_b200.problem import FixedPointConfig
    g = load("fixed_point")
    prob = problem_for(g, name)
    stab = "off" if name.endswith("off") else "spline_upwind"
    res = fixed_point_solve(prob, FixedPointConfig(stabilization=stab, linear_solver="iterative"))
    assert res.iterations == int(g[name + "_it"])
    assert res.gmres_iterations == [int(v) for v in g[name + "_gm"]]
    assert res.pcg_iterations == [int(v) for v in g[name + "_pcg"]]
    for key in ("u", "w"):
        ref = g[name + "_" + key]
        got = getattr(res, key)
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-10, key
    np.testing.assert_allclose(res.increments, g[name + "_inc"], rtol=1e-8)


def pulse_torch(x, t):
    return 1.0 * (x[:, 0] < 0.1).to(x.dtype) * (t < 0.05)


def device_problem_for(g, name):
    from paper_2311_17500_b200.problem import DeviceSource
    prob = problem_for(g, name)
    prob.source = DeviceSource(pulse_source, pulse_torch)
    return prob


@pytest.mark.gpu
@pytest.mark.parametrize("name", SWEEPS)
def test_device_source_load_vector_matches_reference(name):
    """DeviceSource: Gauss-point values evaluated by its torch form and contracted on the GPU."""
    import torch
    from paper_2311_17500_b200.problem import load_vector
    g = load("fixed_point")
    prob = device_problem_for(g, name)
    f = load_vector(prob.space, prob.geometry, prob.source, device=0)
    assert torch.is_tensor(f) and f.is_cuda
    ref = g[name + "_f"]
    assert np.linalg.norm(f.cpu().numpy() - ref) / np.linalg.norm(ref) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["fp_1d_su", "fp_2d_su"])
def test_fixed_point_solve_device_source(name):
    """The driver with a DeviceSource (device load vector + device-resident indicator source)
    reproduces the reference's sweeps, iteration counts and fields."""
    from paper_2311_17500_b200.fixed_point import fixed_point_solve
    from paper_2311_17500_b200.problem import FixedPointConfig
    g = load("fixed_point")
    prob = device_problem_for(g, name)
    res = fixed_point_solve(prob, FixedPointConfig(stabilization="spline_upwind", linear_solver="iterative"))
    assert res.iterations == int(g[name + "_it"])
    assert res.gmres_iterations == [int(v) for v in g[name + "_gm"]]
    for key in ("u", "w"):
        ref = g[name + "_" + key]
        assert np.linalg.norm(getattr(res, key) - ref) / np.linalg.norm(ref) < 1e-10, key


SWEEPS_3D = ["fp_3d_p2_su", "fp_3d_p3_su", "fp_3d_p2_off"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", SWEEPS_3D)
def test_fixed_point_solve_3d_matches_reference(name):
    """3D boxes (p = 2, 3; Spline Upwind and Galerkin): the device driver vs the reference's own
    fixed_point_solve, sweep for sweep (tests/golden/make_golden.py fixed_point_3d)."""
    import os
    from cases import GOLDEN
    from paper_2311_17500_b200.fixed_point import fixed_point_solve
    from paper_2311_17500_b200.problem import FixedPointConfig
    if not os.path.exists(os.path.join(GOLDEN, "fixed_point_3d.npz")):
        pytest.skip("fixture not generated")
    g = load("fixed_point_3d")
    prob = problem_for(g, name, D=float(g[name + "_D"]))
    stab = "off" if name.endswith("off") else "spline_upwind"
    res = fixed_point_solve(prob, FixedPointConfig(stabilization=stab, linear_solver="iterative"))
    assert res.iterations == int(g[name + "_it"])
    assert res.gmres_iterations == [int(v) for v in g[name + "_gm"]]
    assert res.pcg_iterations == [int(v) for v in g[name + "_pcg"]]
    for key in ("u", "w"):
        ref = g[name + "_" + key]
        assert np.linalg.norm(getattr(res, key) - ref) / np.linalg.norm(ref) < 1e-10, key
    np.testing.assert_allclose(res.increments, g[name + "_inc"], rtol=1e-8)
