"""Low-rank geometry / conductivity coefficients on mapped geometries (BASELINE cfg 5: "geometry and
conductivity coefficients low-rank approximated (canonical rank <= 8)").  The
reference integrates the exact pulled-back coefficients (assembly.py:197-219), so there is no reference
output for the approximation itself.  The checks are:

* CP-ALS recovers exactly separable / low-rank arrays;
* the Kronecker-sum factors (geometry.LowRankCoefficients.kron_terms) equal tensor quadrature with the
  reconstructed rank-r coefficient fields -- an identity, checked against the quadrature emulation that
  tests/test_mapped.py pins on the reference's own M_s / K_s (1e-13);
* the low-rank M_s / K_s approach the reference's exact M_s / K_s as the field error does;
* on the GPU, A x equals the oracle Kronecker operator built from the same low-rank factors (1e-12), and
  GMRES / the fixed-point driver reach the exact-coefficient reference solutions to the approximation
  error (the annulus fields are exactly rank 1, so there they match the reference to 1e-10)."""

import numpy as np
import pytest
import torch

from cases import RM
from test_mapped import CASES, FIBRE, assemble_from_tables, load_geo, rel, setup


def band_dense(band, n, p):
    A = np.zeros((n, n))
    for i in range(n):
        for k in range(2 * p + 1):
            j = i - p + k
            if 0 <= j < n:
                A[i, j] = band[i, k]
    return A


def kron_dense(sd, coef, bands, p):
    """Dense N_s x N_s sum_t coef[t] kron_l F_{t,l} (direction d outermost, C order)."""
    n = [s.dimension for s in sd.spaces]
    d = len(n)
    S = 0.0
    for t in range(len(coef)):
        K = np.ones((1, 1))
        for l in reversed(range(d)):
            K = np.kron(K, band_dense(bands[t, l], n[l], p))
        S = S + coef[t] * K
    return S


def test_cp_als_recovers_low_rank_arrays():
    from paper_2311_17500_b200.geometry import cp_als, cp_reconstruct
    g = torch.Generator().manual_seed(3)
    a, b, c = (torch.rand(n, generator=g, dtype=torch.float64) for n in (9, 7, 6))
    X1 = torch.einsum("i,j,k->ijk", a, b, c)
    F, err = cp_als(X1, 1)
    assert err < 1e-13 and torch.allclose(cp_reconstruct(F), X1, rtol=1e-12, atol=0)
    X2 = torch.rand(8, 3, generator=g, dtype=torch.float64) @ torch.rand(3, 11, generator=g, dtype=torch.float64)
    assert cp_als(X2, 2)[1] > 1e-6 and cp_als(X2, 3)[1] < 1e-13            # SVD: optimal truncation
    A = [torch.rand(n, 3, generator=g, dtype=torch.float64) for n in (20, 15, 12)]
    X3 = cp_reconstruct(A)
    errs = [cp_als(X3, r)[1] for r in (1, 2, 3)]
    assert errs[2] < 1e-6 and errs[0] > errs[2]
    assert cp_als(torch.zeros(4, 5, 6, dtype=torch.float64), 2)[1] == 0.0


@pytest.mark.parametrize("name,gkey", CASES)
@pytest.mark.parametrize("fibre", [False, True])
def test_kron_terms_equal_quadrature_with_reconstructed_fields(name, gkey, fibre):
    from paper_2311_17500_b200.geometry import FibreConductivity, MappedSpatialData
    g, geo, st, _ = setup(name, gkey)
    p = st.spatial[0].degree
    cond = FibreConductivity(*FIBRE) if fibre else None
    sd = MappedSpatialData(st.spatial, geo, device=None, conductivity=cond, coefficient_rank=8, coefficient_tol=1e-12)
    lr = sd.lowrank
    d = len(st.spatial)
    nmax = max(s.dimension for s in st.spatial)
    w = sd.wgrid
    M_terms = [(1.0, w * lr.reconstruct("mass"), [(0, 0)] * d)]
    K_terms = [(1.0, w * lr.reconstruct(lr.stiffness_key(a, b)),
                [(1 if l == a else 0, 1 if l == b else 0) for l in range(d)]) for a in range(d) for b in range(d)]
    for kind, terms in (("mass", M_terms), ("stiffness", K_terms)):
        coef, bands = lr.kron_terms(sd, kind, p, nmax)
        S = kron_dense(sd, coef, bands, p)
        Q = assemble_from_tables(sd, terms, p)
        assert rel(S, Q) < 1e-13, kind
        if not fibre:
            # the exact coefficients give the reference's own matrices (fixtures); the low-rank ones
            # are off by at most a small multiple of the fields' CP error
            ref = g[name + ("_M_s" if kind == "mass" else "_K_s")]
            errs = [lr.error["mass"]] if kind == "mass" else [lr.error[k] for k in lr.error if k != "mass"]
            assert rel(S, ref) <= 10 * max(errs) + 1e-13, (kind, rel(S, ref), errs)
    if name == "m2d":
        assert all(r == 1 for r in lr.rank.values())          # the annulus coefficients are separable


def test_coefficient_rank_config_validation():
    from paper_2311_17500_b200.problem import FixedPointConfig
    with pytest.raises(ValueError):
        FixedPointConfig(coefficient_rank=0)


def lowrank_objects(name, gkey, rank=8, tol=1e-12):
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200.geometry import MappedSpatialData
    g, geo, st, _ = setup(name, gkey)
    sd = MappedSpatialData(st.spatial, geo, coefficient_rank=rank, coefficient_tol=tol)
    D = float(g[name + "_D"])
    op = mb.KroneckerOperator(st, 1.0, 1.0, D, RM, spatial_data=sd)
    P = mb.FastDiagPreconditioner.build(st, 1.0, 1.0, D, RM["a"] * RM["c1"], spatial_data=sd, context=op.ctx)
    return g, st, sd, op, P, D


@pytest.mark.gpu
@pytest.mark.parametrize("name,gkey", CASES)
def test_lowrank_operator_matches_kronecker_oracle(name, gkey):
    from oracle.assembly import KronOp, time_factors
    from oracle.splines import make_space_time
    g, st, sd, op, P, D = lowrank_objects(name, gkey)
    p = st.spatial[0].degree
    nmax = max(s.dimension for s in st.spatial)
    Ms = kron_dense(sd, *sd.lowrank.kron_terms(sd, "mass", p, nmax), p)
    Ks = kron_dense(sd, *sd.lowrank.kron_terms(sd, "stiffness", p, nmax), p)
    ost = make_space_time(len(st.spatial), p, [s.dimension - p for s in st.spatial], st.time.dimension - p)
    Wt, Mt = time_factors(ost, 1.0)
    react = RM["a"] * RM["c1"]
    ref = KronOp(st.num_time, st.num_space, [(1.0, Wt, Ms), (D, Mt, Ks), (react, Mt, Ms)])
    x = g[name + "_x"]
    assert rel(op.matvec(x), ref.matvec(x)) < 1e-12
    # against the reference's exact-coefficient operator: the CP error of the fields
    errs = max(sd.lowrank.error.values())
    assert rel(op.matvec(x), g[name + "_y_a"]) <= 10 * errs + 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name,gkey", CASES)
def test_lowrank_gmres_approaches_reference(name, gkey):
    import paper_2311_17500_b200 as mb
    g, st, sd, op, P, D = lowrank_objects(name, gkey)
    x, it, _ = mb.gmres(op, g[name + "_rhs"], precond=P, tol=1e-8, max_iter=400)
    ref_it = int(g[name + "_gm_a_it"])
    errs = max(sd.lowrank.error.values())
    if errs < 1e-13:
        assert it == ref_it and rel(x, g[name + "_gm_a_x"]) < 1e-10
    else:
        assert abs(it - ref_it) <= 2 and rel(x, g[name + "_gm_a_x"]) < 1e3 * errs


@pytest.mark.gpu
def test_lowrank_fixed_point_on_annulus_matches_reference():
    """The annulus coefficients are exactly rank one: the low-rank fixed-point solve (Galerkin) is the
    reference's -- same sweeps, GMRES / PCG counts, u and w to 1e-10 (fixture of
    test_mapped.test_mapped_fixed_point_solve_matches_reference)."""
    from paper_2311_17500_b200.fixed_point import fixed_point_solve
    from paper_2311_17500_b200.problem import FixedPointConfig, MonodomainProblem
    from paper_2311_17500_b200.spaces import SpaceTimeSpace, SplineSpace
    from test_mapped import fixture
    g = fixture()
    st = SpaceTimeSpace([SplineSpace.uniform(2, 8), SplineSpace.uniform(2, 3)], SplineSpace.uniform(2, 8))

    def smooth_source(x, t):
        return np.exp(-((x[:, 0] - 0.3) ** 2 + (x[:, 1] - 0.2) ** 2) / 0.05) * (t < 0.4)

    prob = MonodomainProblem(load_geo("annulus"), st, source=smooth_source, D=1e-3)
    cfg = FixedPointConfig(stabilization="off", linear_solver="iterative", coefficient_rank=8, coefficient_tol=1e-12)
    res = fixed_point_solve(prob, cfg)
    assert res.iterations == int(g["fp_it"])
    assert res.gmres_iterations == [int(v) for v in g["fp_gm"]]
    assert res.pcg_iterations == [int(v) for v in g["fp_pcg"]]
    assert rel(res.u, g["fp_u"]) < 1e-10
    assert rel(res.w, g["fp_w"]) < 1e-10
