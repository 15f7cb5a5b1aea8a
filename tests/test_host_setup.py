"""Host-side factor tables of the product vs the (reference-pinned) oracle.

These are the small 1D/2D tables the kernels consume; the (d+1)-way tensor
work itself is covered by the GPU parity tests.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from cases import CASES, load, oracle_objects
from oracle import stab as ostab
from paper_2311_17500_b200 import factors
from paper_2311_17500_b200.spaces import SpaceTimeSpace, SplineSpace, time_factors


def product_space(g):
    p = int(g["p"])
    return SpaceTimeSpace([SplineSpace.uniform(p, int(n)) for n in g["ne"]],
                          SplineSpace.uniform(p, int(g["ne_t"])))


def dense_su_spatial(st, theta, H, ko):
    """S^s_r[i, j] = sum_k theta[k] prod_l H_l[i_l, j_l-i_l+p, k_l-i_l+ko] (dense, small)."""
    d = len(st.spatial)
    p = st.spatial[0].degree
    n = [s.dimension for s in st.spatial]
    ns = int(np.prod(n))
    idx = np.array(np.unravel_index(np.arange(ns), tuple(reversed(n))))[::-1]  # (d, ns): i_1..i_d
    th = theta
    S = np.zeros((ns, ns))
    for i in range(ns):
        for j in range(ns):
            dj = idx[:, j] - idx[:, i]
            if np.any(np.abs(dj) > p):
                continue
            acc = 0.0
            for k in range(ns):
                dk = idx[:, k] - idx[:, i]
                if np.any(np.abs(dk) > ko):
                    continue
                prod = th[k]
                for l in range(d):
                    prod *= H[l, idx[l, i], dj[l] + p, dk[l] + ko]
                acc += prod
            S[i, j] = acc
    return S


@pytest.mark.parametrize("name", ["case_2d_p2", "case_1d_p1", "case_2d_aniso"])
def test_su_factors_match_oracle(name):
    g = load(name)
    st = product_space(g)
    _, _, _, _, su, lr = oracle_objects(g)
    from paper_2311_17500_b200.operator import Stabilization
    s = Stabilization(st, g["theta"], float(g["su_tol"]), 1.0)
    assert s.rank == lr.rank
    p = st.time.degree
    for r in range(s.rank):
        # time band == C_m s_r sum_k S^t_{r,k}
        T = sum(su[r * p + k][0] * su[r * p + k][1].toarray() for k in range(p))
        band = s.time_bands[r]
        n = T.shape[0]
        Tb = np.zeros_like(T)
        for k in range(2 * p + 1):
            for i in range(n):
                j = i + k - p
                if 0 <= j < n:
                    Tb[i, j] = band[i, k]
        assert np.max(np.abs(Tb - T)) <= 1e-12 * np.max(np.abs(T))
        # spatial factor up to the SVD sign: compare theta-weighted stencils
        Ss = su[r * p][2].toarray()
        sign = np.sign(np.dot(s.theta[r], lr.space_factors[:, r]))
        S = dense_su_spatial(st, sign * s.theta[r], s.H, s.ko)
        assert np.max(np.abs(S - Ss)) <= 1e-12 * np.max(np.abs(Ss))


def test_upwind_weights_match_oracle():
    from oracle.splines import Space
    for p, ne in ((1, 4), (2, 5), (3, 6), (3, 9)):
        tau_o = ostab.compute_tau(Space.uniform(p, ne))
        tau_p = factors.upwind_weights(SplineSpace.uniform(p, ne))
        x = np.linspace(0, 1, 23)
        for k in range(1, p + 1):
            a, b = tau_p.evaluate(k, x), tau_o.evaluate(k, x)
            assert np.max(np.abs(a - b)) <= 1e-9 * max(np.max(np.abs(b)), 1e-30)


@pytest.mark.parametrize("name", CASES)
def test_real_pencil_fd_apply_matches_reference(name):
    """numpy evaluation of the REAL-block P^-1 == reference complex P^-1 (golden)."""
    g = load(name)
    st = product_space(g)
    d = len(st.spatial)
    pen = factors.time_pencil(st, float(g["T"]))
    eigs = factors.spatial_eigs(st)
    sig = np.atleast_1d(g["sigma"])
    sig = np.repeat(sig, d) if sig.size == 1 else sig
    mu = np.zeros(st.spatial_shape)
    for l in range(d):
        shp = [1] * d
        shp[d - 1 - l] = -1
        mu = mu + sig[l] * eigs[l][1].reshape(shp)
    mu = mu.ravel() + 0.13 * 0.26

    def mode(A, X, ax):
        t = np.moveaxis(X, ax, 0)
        o = (A @ t.reshape(t.shape[0], -1)).reshape((A.shape[0],) + t.shape[1:])
        return np.moveaxis(o, 0, ax)

    Y = mode(pen.Q.T, g["x"].reshape(st.coeff_shape), 0)
    for l in range(d):
        Y = mode(eigs[l][0].T, Y, 1 + (d - 1 - l))
    Y = Y.reshape(st.num_time, -1)
    diag, off, part = pen.coupling()
    a = diag[:, None] + mu[None]
    e = diag[part][:, None] + mu[None]
    b = off[:, None]
    c = off[part][:, None]
    det = a * e - b * c

    def Dinv(v):
        return (e * v - b * v[part]) / det

    gb = pen.g[:, None] * np.ones_like(mu)[None]
    dy, db = Dinv(Y[:-1]), Dinv(gb)
    xl = (Y[-1] - np.sum(pen.g_low[:, None] * dy, 0)) / (pen.sigma + mu - np.sum(pen.g_low[:, None] * db, 0))
    Z = np.vstack([dy - db * xl[None], xl[None]]).reshape(st.coeff_shape)
    Z = mode(pen.Q, Z, 0)
    for l in range(d):
        Z = mode(eigs[l][0], Z, 1 + (d - 1 - l))
    ref = g["z_pc"]
    assert np.linalg.norm(Z.ravel() - ref) / np.linalg.norm(ref) < 1e-12
    # Q^T M_t Q = I
    Wt, Mt = time_factors(st, float(g["T"]))
    assert np.max(np.abs(pen.Q.T @ Mt @ pen.Q - np.eye(st.num_time))) < 1e-10


def test_lowrank_gram_path_matches_svd(monkeypatch):
    """Large wide indicators use the Gram eigendecomposition: same rank, same singular values,
    same truncated reconstruction as numpy's SVD (to the truncation's own rounding sensitivity)."""
    import numpy as np
    import paper_2311_17500_b200.factors as F
    rng = np.random.default_rng(3)
    nt, ns = 40, 4000
    tg = np.linspace(0, 1, nt)[:, None]
    xs = np.linspace(0, 1, ns)[None, :]
    th = np.clip(np.exp(-((xs - 0.2 - 0.5 * tg) / 0.08) ** 2) + 0.05 * rng.uniform(0, 1, (nt, ns)), 0, 1)
    ref = F.lowrank_factorize(th, 0.1)
    monkeypatch.setattr(F, "GRAM_MIN_SIZE", 0)
    got = F.lowrank_factorize(th, 0.1)
    assert got.rank == ref.rank
    np.testing.assert_allclose(got.weights, ref.weights, rtol=1e-12)
    A = (ref.time_factors * ref.weights) @ ref.space_factors.T
    B = (got.time_factors * got.weights) @ got.space_factors.T
    assert np.abs(A - B).max() <= 1e-10 * np.abs(A).max()
