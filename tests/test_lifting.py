"""u0 lifting (nonzero initial data, absent in the reference).

CPU: the oracle extension (oracle/lifting.py) reduces to the reference on the reference's own
fixtures, and the host lifting tables equal the oracle's full time factors.  GPU: the device lifted
operator, its right-hand side correction, the lifted indicator and whole fixed-point solves with the
BASELINE stimuli against the oracle extension (equal sweeps and GMRES / PCG counts, u and w <= 1e-10).
"""

import numpy as np
import pytest
import scipy.sparse as sp

from cases import RM, load, oracle_objects, space_of


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", ["case_3d_p3", "case_2d_aniso", "case_1d_p1"])
def test_oracle_full_time_blocks_reduce_to_reference(name):
    """The full-time M_R and SU factors of the oracle extension: with a zero lifted slab their
    constrained blocks are the reference's (golden y_mr and y_a - y_sep)."""
    from oracle import lifting
    from oracle import stab as ostab
    g = load(name)
    st = space_of(g)
    ns = st.num_space
    T = float(g["T"])
    MRf = lifting.reaction_mass_full(st, T, RM, lifting.full_coeffs(st, g["u"], None),
                                     lifting.full_coeffs(st, g["w"], None))
    assert rel(MRf[ns:, ns:] @ g["x"], g["y_mr"]) < 1e-13
    _, _, _, _, _, lr = oracle_objects(g)
    tau = ostab.compute_tau(st.time)
    X = g["x"].reshape(st.num_time, ns)
    y = np.zeros_like(X)
    for c, St, Ss in lifting.su_full_terms(tau, lr, st, 1.0):
        y += c * np.asarray(Ss @ (St[1:, 1:] @ X).T).T
    assert rel(y.ravel(), g["y_a"] - g["y_sep"]) < 1e-12


@pytest.mark.parametrize("p", [1, 2, 3])
def test_host_lift_columns_match_oracle(p):
    """spaces.time_lift_columns and factors.su_time_lift = column 0 of the oracle's full time factors."""
    from oracle import lifting
    from oracle import stab as ostab
    from oracle.splines import make_space_time
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200.factors import su_time_lift
    from paper_2311_17500_b200.spaces import time_lift_columns
    ost = make_space_time(2, p, (4, 3), 6)
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, n) for n in (4, 3)], mb.SplineSpace.uniform(p, 6))
    Wf, Mf = lifting.full_time_factors(ost, 1.7)
    wcol, mcol = time_lift_columns(st, 1.7)
    np.testing.assert_allclose(wcol, Wf[1:, 0].toarray().ravel(), atol=1e-15)
    np.testing.assert_allclose(mcol, Mf[1:, 0].toarray().ravel(), atol=1e-15)
    th = np.random.default_rng(p).random((st.num_time, st.num_space))
    stab = mb.Stabilization(st, th, 0.3, 1.3)
    lr = ostab.lowrank_factorize(ostab.indicator_for(ost, th), 0.3)
    assert stab.rank == lr.rank
    ref = np.zeros((lr.rank, st.num_time))
    tau = ostab.compute_tau(ost.time)
    for i, (c, St, _) in enumerate(lifting.su_full_terms(tau, lr, ost, 1.3)):
        ref[i // p] += c * St[1:, 0].toarray().ravel()
    np.testing.assert_allclose(su_time_lift(st, stab.tau, stab.lowrank, 1.3), ref, rtol=1e-12, atol=1e-14)


def u0_step(x):
    """BASELINE cfg 1 stimulus: u0 = 1 on x < 0.1."""
    return 1.0 * (x[:, 0] < 0.1)


def u0_corner(x):
    """BASELINE cfg 2 stimulus: u0 = 1 on the corner square [0, 0.1]^2."""
    return 1.0 * (x[:, 0] < 0.1) * (x[:, 1] < 0.1)


def u0_smooth(x):
    return np.exp(-np.sum((x - 0.3) ** 2, axis=1) / 0.05)


def test_lift_coefficients_are_the_greville_quasi_interpolant():
    import paper_2311_17500_b200 as mb
    from oracle import lifting
    from oracle.splines import Space
    from paper_2311_17500_b200.problem import BoxGeometry, MonodomainProblem, lift_coefficients
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(2, 9), mb.SplineSpace.uniform(3, 5)], mb.SplineSpace.uniform(2, 4))
    prob = MonodomainProblem(BoxGeometry([1.0, 1.0], 1.0), st, u0=u0_smooth)
    c = lift_coefficients(prob)
    np.testing.assert_allclose(c, lifting.greville_lift([Space.uniform(2, 9), Space.uniform(3, 5)], u0_smooth),
                               rtol=1e-14)
    assert lift_coefficients(MonodomainProblem(BoxGeometry([1.0, 1.0], 1.0), st)) is None


# ---------------------------------------------------------------------------------------------- GPU
def _device_op(st, T, D, u=None, w=None, theta=None, lift=None):
    import paper_2311_17500_b200 as mb
    stab = None if theta is None else mb.Stabilization(st, theta, 0.3, 1.0)
    return mb.KroneckerOperator(st, T, 1.0, D, RM, u=u, w=w, stabilization=stab, lift=lift)


def _oracle_lifted(ost, T, D, u, w, theta, lift):
    """Oracle operator (constrained block) and lifted column applied to the lift (oracle/lifting)."""
    from oracle import assembly as asm
    from oracle import lifting
    from oracle import stab as ostab
    ns = ost.num_space
    Wf, Mf = lifting.full_time_factors(ost, T)
    sig = np.atleast_1d(D)
    Ms, Ks = asm.box_spatial(ost.spatial, diffusion=None if sig.size == 1 else sig)
    Dk = float(sig[0]) if sig.size == 1 else 1.0
    terms = [(1.0, Wf, Ms), (Dk, Mf, Ks)]
    if theta is not None:
        lr = ostab.lowrank_factorize(ostab.indicator_for(ost, theta), 0.3)
        terms += lifting.su_full_terms(ostab.compute_tau(ost.time), lr, ost, 1.0)
    MRf = lifting.reaction_mass_full(ost, T, RM, lifting.full_coeffs(ost, u, lift), lifting.full_coeffs(ost, w, None))
    op = asm.KronOp(ost.num_time, ns, [(c, sp.csr_matrix(Tm[1:, 1:]), S) for c, Tm, S in terms],
                    sp.csr_matrix(MRf[ns:, ns:]))
    corr = sum(c * np.kron(Tm[1:, 0].toarray().ravel(), S @ lift) for c, Tm, S in terms) + MRf[ns:, :ns] @ lift
    return op, corr


@pytest.mark.gpu
@pytest.mark.parametrize("d,p,su", [(1, 2, True), (2, 3, True), (3, 2, False), (3, 3, True)])
def test_lifted_operator_and_correction(d, p, su):
    """A at a general iterate with the lifted reaction, and A_{c,0} u0, vs the oracle extension."""
    import paper_2311_17500_b200 as mb
    from oracle.splines import make_space_time
    nes = {1: (9,), 2: (5, 4), 3: (3, 2, 4)}[d]
    ne_t, T, D = 5, 1.3, 2e-2
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, n) for n in nes], mb.SplineSpace.uniform(p, ne_t))
    ost = make_space_time(d, p, nes, ne_t)
    rng = np.random.default_rng(10 * d + p)
    N, ns = st.num_dof, st.num_space
    u, w, x = rng.uniform(0, 1, N), rng.uniform(0, 0.1, N), rng.uniform(-1, 1, N)
    lift = rng.uniform(0, 1, ns)
    theta = rng.random((st.num_time, ns)) if su else None
    op = _device_op(st, T, D, u, w, theta, lift)
    oop, corr = _oracle_lifted(ost, T, D, u, w, theta, lift)
    for store in (0, 1):
        from paper_2311_17500_b200 import _lib
        _lib.call("mi_op_set_reaction_store", op.ctx.handle, store)
        assert rel(op.matvec(x), oop.matvec(x)) < 1e-12
        assert rel(op.lift_apply().cpu().numpy(), corr) < 1e-12
    # zero iterate: the lifted field is u0 b_0, so the reaction is M_R(u0 b_0, 0), not a c1 M (x) M
    op0 = _device_op(st, T, D, None, None, theta, lift)
    oop0, corr0 = _oracle_lifted(ost, T, D, np.zeros(N), np.zeros(N), theta, lift)
    assert not op0.zero_iterate
    assert rel(op0.matvec(x), oop0.matvec(x)) < 1e-12
    assert rel(op0.lift_apply().cpu().numpy(), corr0) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("d,p", [(1, 2), (2, 3), (3, 2)])
def test_lifted_indicator(d, p):
    """Device compute_theta of the lifted field vs oracle/lifting.compute_theta."""
    import paper_2311_17500_b200 as mb
    from oracle import lifting
    from oracle.splines import make_space_time
    from paper_2311_17500_b200.problem import BoxGeometry, MonodomainProblem
    from paper_2311_17500_b200.theta import DeviceIndicator
    nes = {1: (11,), 2: (6, 5), 3: (4, 3, 3)}[d]
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, n) for n in nes], mb.SplineSpace.uniform(p, 6))
    ost = make_space_time(d, p, nes, 6)
    prob = MonodomainProblem(BoxGeometry([1.0] * d, 1.5), st, D=2e-2)
    rng = np.random.default_rng(d)
    u, w = rng.uniform(0, 1, st.num_dof), rng.uniform(0, 0.1, st.num_dof)
    lift = rng.uniform(0, 1, st.num_space)
    got = DeviceIndicator(prob).compute(u, w, lift=lift).values
    ref = lifting.compute_theta(ost, 1.5, 1.0, 2e-2, RM, None, u, w, lift)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-14)
    # the lifted field alone (zero iterate): a nonzero denominator from u0 b_0
    z = np.zeros(st.num_dof)
    got = DeviceIndicator(prob).compute(z, z, lift=lift).values
    np.testing.assert_allclose(got, lifting.compute_theta(ost, 1.5, 1.0, 2e-2, RM, None, z, z, lift),
                               rtol=1e-12, atol=1e-14)


FP_CASES = [
    # BASELINE cfg 1 exactly: 1D p=2 64 x 64, D = 1e-3, u0 = 1 on x < 0.1, Spline Upwind, GMRES rtol 1e-8
    ("cfg1", 1, 2, (64,), 64, 1e-3, u0_step, "spline_upwind"),
    ("cfg1_galerkin", 1, 2, (64,), 64, 1e-3, u0_step, "off"),
    # cfg 2's corner-square stimulus on a reduced 2D p=3 mesh
    ("corner_2d", 2, 3, (10, 10), 12, 1e-3, u0_corner, "spline_upwind"),
    # cfg 3's planar stimulus, anisotropic sigma, on a reduced 3D p=2 mesh
    ("planar_3d", 3, 2, (6, 5, 4), 6, (1e-3, 4e-4, 4e-4), lambda x: 1.0 * (x[:, 0] < 0.05), "spline_upwind"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,d,p,nes,ne_t,D,u0,stab", FP_CASES, ids=[c[0] for c in FP_CASES])
def test_lifted_fixed_point_matches_oracle(name, d, p, nes, ne_t, D, u0, stab):
    """The device fixed-point driver on the lifted problem vs oracle/lifting.fixed_point_solve:
    equal sweeps, GMRES and PCG counts per sweep, u and w <= 1e-10."""
    import paper_2311_17500_b200 as mb
    from oracle import lifting
    from oracle.splines import make_space_time
    from paper_2311_17500_b200.problem import BoxGeometry
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, n) for n in nes], mb.SplineSpace.uniform(p, ne_t))
    prob = mb.MonodomainProblem(BoxGeometry([1.0] * d, 1.0), st, D=D, u0=u0)
    res = mb.fixed_point_solve(prob, mb.FixedPointConfig(stabilization=stab, linear_solver="iterative"))
    ost = make_space_time(d, p, nes, ne_t)
    ref = lifting.fixed_point_solve(ost, 1.0, D, RM, u0=u0, stabilization=stab)
    assert res.converged and ref["converged"]
    np.testing.assert_allclose(res.lift, ref["lift"], rtol=0, atol=0)
    assert res.iterations == ref["iterations"]
    assert res.gmres_iterations == ref["gmres"]
    assert res.pcg_iterations == ref["pcg"]
    assert rel(res.u, ref["u"]) < 1e-10
    assert rel(res.w, ref["w"]) < 1e-10
    np.testing.assert_allclose(res.increments, ref["increments"], rtol=1e-8)


@pytest.mark.gpu
@pytest.mark.parametrize("d,p", [(1, 2), (2, 3), (3, 2)])
def test_recovery_solver_matches_solve_w_system(d, p):
    """wsolve.RecoverySolver (device) vs the restatement of solve_w_system + pcg +
    KroneckerMassPreconditioner (linalg.py:176-203, 450-547): w to 1e-12 and equal PCG counts."""
    import paper_2311_17500_b200 as mb
    from oracle import assembly as asm
    from oracle import lifting
    from oracle.splines import make_space_time
    from paper_2311_17500_b200.wsolve import RecoverySolver
    nes = {1: (13,), 2: (6, 5), 3: (4, 3, 5)}[d]
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, n) for n in nes], mb.SplineSpace.uniform(p, 7))
    ost = make_space_time(d, p, nes, 7)
    g = np.random.default_rng(d).standard_normal(st.num_dof)
    w, its = RecoverySolver(st, 1.3, 0.013, 1.0, 1e-8).solve(g)
    Wt, Mt = asm.time_factors(ost, 1.3)
    Ms, _ = asm.box_spatial(ost.spatial)
    wr, itr = lifting.solve_w(ost, Wt, Mt, Ms, 0.013, 1.0, g, 1e-8)
    assert list(its) == list(itr)
    assert rel(w, wr) < 1e-12
