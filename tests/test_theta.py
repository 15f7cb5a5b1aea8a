"""Spline Upwind residual indicator (compute_theta, stabilization.py:235-339):
host restatement (CPU) and the device kernels (GPU) vs the reference's own
values on equal-degree spaces (tests/golden/theta.npz, make_golden.py theta)."""

import numpy as np
import pytest

from cases import load

CASES = ["th3d", "th1d"]


def pulse_source(x, t):
    return 1.0 * (x[:, 0] < 0.1) * (t < 0.05)


def problem_for(g, name):
    import paper_2311_17500_b200.spaces as sp
    from paper_2311_17500_b200.problem import BoxGeometry, MonodomainProblem
    p = int(g[name + "_p"])
    st = sp.SpaceTimeSpace([sp.SplineSpace.uniform(p, int(n)) for n in g[name + "_ne"]],
                           sp.SplineSpace.uniform(p, int(g[name + "_ne_t"])))
    src = pulse_source if int(g[name + "_src"]) else None
    return MonodomainProblem(BoxGeometry(g[name + "_L"], float(g[name + "_T"])), st, source=src,
                             D=float(g[name + "_D"]))


@pytest.mark.parametrize("name", CASES)
def test_host_theta_matches_reference(name):
    from paper_2311_17500_b200.problem import host_compute_theta as compute_theta
    g = load("theta")
    prob = problem_for(g, name)
    th = compute_theta(prob, g[name + "_u"], g[name + "_w"])
    np.testing.assert_allclose(th.values, g[name + "_values"], rtol=1e-12, atol=1e-14)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("chunk", [1 << 26, 500])
def test_device_theta_matches_reference(name, chunk):
    from paper_2311_17500_b200.theta import DeviceIndicator
    g = load("theta")
    prob = problem_for(g, name)
    di = DeviceIndicator(prob, chunk_points=chunk)
    th = di.compute(g[name + "_u"], g[name + "_w"])
    np.testing.assert_allclose(th.values, g[name + "_values"], rtol=1e-12, atol=1e-14)
    assert th.values.shape == g[name + "_values"].shape


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("chunk", [1 << 26, 500])
def test_device_theta_device_source(name, chunk):
    """The source given as a DeviceSource: its Gauss values are evaluated on the GPU."""
    from paper_2311_17500_b200.problem import DeviceSource
    from paper_2311_17500_b200.theta import DeviceIndicator
    g = load("theta")
    prob = problem_for(g, name)
    if prob.source is not None:
        prob.source = DeviceSource(pulse_source, lambda x, t: 1.0 * (x[:, 0] < 0.1).to(x.dtype) * (t < 0.05))
    th = DeviceIndicator(prob, chunk_points=chunk).compute(g[name + "_u"], g[name + "_w"])
    np.testing.assert_allclose(th.values, g[name + "_values"], rtol=1e-12, atol=1e-14)


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 2, 3])
def test_device_theta_matches_host_2d(p):
    import paper_2311_17500_b200.spaces as sp
    from paper_2311_17500_b200.problem import BoxGeometry, MonodomainProblem, host_compute_theta as compute_theta
    from paper_2311_17500_b200.theta import DeviceIndicator
    st = sp.SpaceTimeSpace([sp.SplineSpace.uniform(p, 7), sp.SplineSpace.uniform(p, 4)], sp.SplineSpace.uniform(p, 5))
    prob = MonodomainProblem(BoxGeometry([2.0, 0.7], 1.5), st, source=pulse_source, D=3e-2)
    rng = np.random.default_rng(p)
    u = rng.uniform(-0.2, 1.1, st.num_dof)
    w = rng.uniform(0, 0.2, st.num_dof)
    ref = compute_theta(prob, u, w).values
    got = DeviceIndicator(prob).compute(u, w).values
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-14)


@pytest.mark.gpu
def test_device_theta_zero_denominator():
    """u = w = 0 with a source: denominator 0, stabilizer switched fully on where the residual is hot
    (stabilization.py:317-333), with the reference's warning."""
    import paper_2311_17500_b200.spaces as sp
    from paper_2311_17500_b200.problem import BoxGeometry, MonodomainProblem, host_compute_theta as compute_theta
    from paper_2311_17500_b200.theta import DeviceIndicator
    st = sp.SpaceTimeSpace([sp.SplineSpace.uniform(2, 12)], sp.SplineSpace.uniform(2, 10))
    prob = MonodomainProblem(BoxGeometry([1.0], 1.0), st, source=pulse_source, D=1e-3)
    z = np.zeros(st.num_dof)
    with pytest.warns(RuntimeWarning):
        ref = compute_theta(prob, z, z).values
    with pytest.warns(RuntimeWarning):
        got = DeviceIndicator(prob).compute(z, z).values
    np.testing.assert_array_equal(got, ref)
    assert got.max() == 1.0


@pytest.mark.gpu
def test_device_theta_anisotropic_matches_host():
    """Diagonal anisotropic D (cfg 3's sigma; SURVEY App. B extension): device vs host restatement."""
    import paper_2311_17500_b200.spaces as sp
    from paper_2311_17500_b200.problem import BoxGeometry, MonodomainProblem, host_compute_theta as compute_theta
    from paper_2311_17500_b200.theta import DeviceIndicator
    st = sp.SpaceTimeSpace([sp.SplineSpace.uniform(2, n) for n in (5, 4, 3)], sp.SplineSpace.uniform(2, 4))
    prob = MonodomainProblem(BoxGeometry([1.0, 0.8, 1.2], 1.0), st, source=pulse_source, D=[1e-1, 4e-2, 2e-2])
    rng = np.random.default_rng(5)
    u = rng.uniform(0, 1, st.num_dof)
    w = rng.uniform(0, 0.1, st.num_dof)
    ref = compute_theta(prob, u, w).values
    got = DeviceIndicator(prob).compute(u, w).values
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-14)
