"""Fast-diagonalisation preconditioner -- oracle restatement of linalg.py:75-356.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from .assembly import time_factors


class ConsistencyError(RuntimeError):
    pass


class DecompositionError(RuntimeError):
    pass


def _dense(A):
    return A.toarray() if sp.issparse(A) else np.asarray(A, float)


def gen_eig(K, M):
    """linalg.py:75-89: eigh(K, M) -> (U, lam), U^T M U = I."""
    lam, U = sla.eigh(_dense(K), _dense(M))
    return U, lam


class Pencil:
    """linalg.py:92-124 data of the bordered time pencil."""

    def __init__(self, U, lam, g, sigma, W):
        self.U_full, self.eigenvalues, self.g, self.sigma, self.W = U, lam, g, sigma, W


def time_pencil(Wt, Mt, cond_limit=1e12):
    """linalg.py:127-173: Cholesky-whitened skew interior + border column."""
    W, M = _dense(Wt), _dense(Mt)
    n = W.shape[0]
    Wi, Mi, wb, mb = W[:-1, :-1], M[:-1, :-1], W[:-1, -1], M[:-1, -1]
    L = sla.cholesky(Mi, lower=True)
    S = sla.solve_triangular(L, Wi, lower=True)
    S = sla.solve_triangular(L, S.T, lower=True).T
    S = 0.5 * (S - S.T)
    mu, Q = sla.eigh(1j * S)
    lam = -1j * mu
    Ui = sla.solve_triangular(L.T, Q, lower=False)
    v = sla.cho_solve((L, True), -mb)
    s = float(v @ Mi @ v + 2.0 * (v @ mb) + M[-1, -1])
    if s <= 0:
        raise DecompositionError("temporal mass matrix not positive definite")
    t, rho = v / np.sqrt(s), 1.0 / np.sqrt(s)
    U = np.zeros((n, n), dtype=complex)
    U[:-1, :-1] = Ui
    U[:-1, -1] = t
    U[-1, -1] = rho
    g = Ui.conj().T @ (Wi @ t + rho * wb)
    tr = np.concatenate([t, [rho]])
    sigma = complex(tr.conj() @ (W @ tr))
    if np.linalg.cond(U) > cond_limit:
        raise DecompositionError("temporal pencil eigenvectors ill-conditioned")
    return Pencil(U, lam, g, sigma, W)


def _mode(mat, X, axis):
    t = np.moveaxis(X, axis, 0)
    out = (mat @ t.reshape(t.shape[0], -1)).reshape((mat.shape[0],) + t.shape[1:])
    return np.moveaxis(out, 0, axis)


class FastDiag:
    """linalg.py:206-356 for boxes (unit separable weights).

    ``lam_s`` is the flattened spatial eigenvalue grid; for the anisotropic
    extension pass sum_l sigma_l lam_l with diffusion=1.
    """

    def __init__(self, eigs, lam_s, pencil, cm, diff, react):
        self.eigs, self.lam_s, self.pencil = eigs, np.asarray(lam_s, float), pencil
        self.cm, self.diff, self.react = float(cm), float(diff), float(react)
        self.nt = pencil.U_full.shape[0]
        self.ns = self.lam_s.size
        self.shape_c = (self.nt,) + tuple(U.shape[0] for U, _ in reversed(eigs))

    @classmethod
    def build(cls, st, T, cm, diff, react, sigma=None, lengths=None):
        """linalg.py:264-307 with ``spatial_data`` of a box (solver.py:193-202).

        For a box with side lengths L the separable weights of linalg.py:228-262
        are constants: mass_l = det^(1/d), stiff_l = det^(1/d) / L_l^2.
        """
        d = st.d
        L = np.ones(d) if lengths is None else np.asarray(lengths, float)
        cmass = np.prod(L) ** (1.0 / d)
        eigs = []
        for l, s in enumerate(st.spatial):
            M, K, _ = _weighted_mk(s, cmass, cmass / L[l] ** 2)
            eigs.append(gen_eig(K, M))
        grid = np.zeros(st.spatial_shape)
        for l in range(d):
            shp = [1] * d
            shp[d - 1 - l] = eigs[l][1].size
            f = 1.0 if sigma is None else sigma[l]
            grid = grid + f * eigs[l][1].reshape(shp)
        Wt, Mt = time_factors(st, T)
        return cls(eigs, grid.ravel(), time_pencil(Wt, Mt), cm, 1.0 if sigma is not None else diff, react)

    def blocks(self):
        """linalg.py:309-315."""
        base = self.diff * self.lam_s + self.react
        Hi = self.cm * self.pencil.eigenvalues[:, None] + base[None, :]
        Hl = self.cm * self.pencil.sigma + base
        B = self.cm * self.pencil.g[:, None]
        return Hi, Hl, B

    def apply(self, r):
        """linalg.py:317-353."""
        r = np.asarray(r, float).ravel()
        if r.size != self.nt * self.ns:
            raise ValueError("dimension mismatch in preconditioner application")
        d = len(self.eigs)
        X = r.reshape(self.shape_c).astype(complex)
        X = _mode(self.pencil.U_full.conj().T, X, 0)
        for l in range(d):
            X = _mode(self.eigs[l][0].T, X, 1 + (d - 1 - l))
        Y = X.reshape(self.nt, self.ns)
        Hi, Hl, B = self.blocks()
        yi, yl = Y[:-1], Y[-1]
        den = Hl + np.sum(np.abs(B) ** 2 / Hi, axis=0)
        xl = (yl + np.sum(np.conj(B) * yi / Hi, axis=0)) / den
        xi = (yi - B * xl[None, :]) / Hi
        Z = np.vstack([xi, xl[None, :]]).reshape(self.shape_c)
        Z = _mode(self.pencil.U_full, Z, 0)
        for l in range(d):
            Z = _mode(self.eigs[l][0], Z, 1 + (d - 1 - l))
        f = Z.ravel()
        sc = np.max(np.abs(f.real), initial=0.0)
        if sc > 0 and np.max(np.abs(f.imag)) > 1e-8 * sc:
            raise ConsistencyError("preconditioner produced a non-negligible imaginary part")
        return f.real.copy()

    __call__ = apply


def _weighted_mk(space, cm=1.0, ck=1.0):
    """The solver always passes spatial_data (solver.py:193-202), so the
    weighted univariate path with unit weights and a p+1 rule on the spatial
    quadrature grid is used (linalg.py:296-299: ``rule=spatial_data.rules[l]``
    is the default q=p+1 rule).  Identical to the unweighted factors on boxes.
    """
    from .assembly import Rule, gram
    rule = Rule.on(space)
    one = np.ones(rule.points.size)
    return gram(space, 0, 0, cm * one, rule), gram(space, 1, 1, ck * one, rule), None
