"""Spline Upwind stabiliser: upwind weights, low-rank indicator, Kronecker terms.

Oracle restatement of monoiga/stabilization.py (the parts the solve uses).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import numpy as np
import scipy.sparse as sp
from scipy.interpolate import RegularGridInterpolator

from .assembly import Rule, kron_list, spatial_colloc, weight_grid
from .splines import Space


def _max_smooth_knots(bp, p):
    """stabilization.py:38-42."""
    return np.concatenate([np.zeros(p + 1), np.asarray(bp, float)[1:-1], np.ones(p + 1)])


class UpwindWeights:
    """stabilization.py:45-81: tau_k as splines of degree p-k (parametric)."""

    def __init__(self, spaces, coeffs, residual):
        self.spaces = spaces
        self.coeffs = coeffs
        self.residual = residual

    def evaluate(self, k, pts):
        C = self.spaces[k - 1].colloc(np.asarray(pts, float), 0)
        return np.asarray(C @ self.coeffs[k - 1]).ravel()


def compute_tau(tspace):
    """stabilization.py:84-145: column-equilibrated least squares for tau_k."""
    p = tspace.degree
    spaces = [Space(_max_smooth_knots(tspace.breakpoints, p - k), p - k) for k in range(1, p + 1)]
    rule = Rule.on(tspace, 2 * p)
    x, w = rule.points, rule.weights
    B = [tspace.colloc(x, k).toarray() for k in range(p + 1)]
    Phi = [s.colloc(x, 0).toarray() for s in spaces]
    off = np.concatenate([[0], np.cumsum([s.dimension for s in spaces])])
    n = tspace.dimension
    G, b = [], []
    for i in range(n - 1):
        for ell in range(1, min(p, n - 1 - i) + 1):
            j = i + ell
            row = np.concatenate([(w * B[k][:, j] * B[k][:, i]) @ Phi[k - 1] for k in range(1, p + 1)])
            G.append(row)
            b.append(-np.sum(w * B[1][:, j] * B[0][:, i]))
    G, b = np.array(G), np.array(b)
    cn = np.linalg.norm(G, axis=0)
    cn[cn == 0.0] = 1.0
    sol = np.linalg.lstsq(G / cn, b, rcond=None)[0] / cn
    res = np.max(np.abs(G @ sol - b)) / max(np.max(np.abs(b)), 1e-300)
    if res > 1e-8:
        raise RuntimeError("upwind weight conditions not satisfied (residual %.3e)" % res)
    return UpwindWeights(spaces, [sol[off[k]:off[k + 1]] for k in range(p)], res)


class Indicator:
    """stabilization.py:177-193: N_t x N_s indicator on the Greville grids."""

    def __init__(self, values, tgrev, sgrevs, sshape):
        self.values = np.asarray(values, float)
        self.time_greville = np.asarray(tgrev, float)
        self.spatial_grevilles = [np.asarray(g, float) for g in sgrevs]
        self.spatial_shape = tuple(sshape)


def indicator_for(st, values):
    return Indicator(values, st.time_greville(), [s.greville() for s in st.spatial], st.spatial_shape)


class LowRank:
    """stabilization.py:342-398: truncated SVD + piecewise-linear profiles."""

    def __init__(self, ind, rank, Ut, Vs, s, tol):
        self.indicator, self.rank = ind, int(rank)
        self.time_factors, self.space_factors, self.weights, self.tol = Ut, Vs, s, tol

    def time_profile(self, r, pts):
        return np.interp(np.asarray(pts, float), self.indicator.time_greville, self.time_factors[:, r])

    def space_profile(self, r, axes):
        g = self.indicator.spatial_grevilles
        d = len(g)
        coords = tuple(g[l] for l in reversed(range(d)))
        vals = self.space_factors[:, r].reshape(self.indicator.spatial_shape)
        f = RegularGridInterpolator(coords, vals, method="linear", bounds_error=False, fill_value=None)
        mesh = np.meshgrid(*[axes[l] for l in reversed(range(d))], indexing="ij")
        pts = np.stack([m.ravel() for m in mesh], axis=-1)
        pts = np.clip(pts, [c[0] for c in coords], [c[-1] for c in coords])
        return f(pts).reshape(mesh[0].shape)


def lowrank_factorize(ind, tol):
    """stabilization.py:401-418: smallest rank with tail <= tol * ||Theta||_F."""
    th = ind.values
    nrm = np.linalg.norm(th)
    if nrm == 0.0:
        nt, ns = th.shape
        return LowRank(ind, 0, np.zeros((nt, 0)), np.zeros((ns, 0)), np.zeros(0), tol)
    U, s, Vt = np.linalg.svd(th, full_matrices=False)
    tail = np.sqrt(np.concatenate([np.cumsum(s[::-1] ** 2)[::-1], [0.0]]))
    r = max(int(np.argmax(tail <= tol * nrm)), 1)
    return LowRank(ind, r, U[:, :r], Vt[:r].T.copy(), s[:r].copy(), tol)


def assemble_stabilization(tau, lr, st, capacitance, lengths=None):
    """stabilization.py:448-489 -> list of Kronecker terms (439-445).

    Returns [(C_m s_r, S^t_{r,k}, S^s_r) for r, k] exactly as
    ``StabilizationMatrices.terms`` orders them.
    """
    p = st.time.degree
    if lr.rank == 0:
        return []
    tr = Rule.on(st.time, p + 2, lr.indicator.time_greville)
    tx, tw = tr.points, tr.weights
    tauv = [tau.evaluate(k, tx) for k in range(1, p + 1)]
    tcol = [st.time_colloc(tx, k) for k in range(1, p + 1)]
    qs = max(s.degree for s in st.spatial) + 2
    rules, scols = spatial_colloc(st.spatial, qs, lr.indicator.spatial_grevilles)
    C = kron_list([scols[l] for l in reversed(range(st.d))])
    wg = weight_grid(rules, lengths)
    axes = [r.points for r in rules]
    out = []
    for r in range(lr.rank):
        prof_t = lr.time_profile(r, tx)
        Ss = sp.csr_matrix(C.T @ sp.diags((wg * lr.space_profile(r, axes)).ravel()) @ C)
        coef = capacitance * lr.weights[r]
        for k in range(1, p + 1):
            Ck = tcol[k - 1]
            St = sp.csr_matrix(Ck.T @ sp.diags(tw * tauv[k - 1] * prof_t) @ Ck)
            out.append((coef, St, Ss))
    return out
