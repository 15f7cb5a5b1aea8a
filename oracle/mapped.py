"""Mapped (non-affine) geometries: the spline map, pulled-back quadrature mass and
stiffness, and the separable preconditioner weights.

Oracle restatement of monoiga/geometry.py:31-214 (GeometryMap.grid_data,
jacobian_inverse_and_det), monoiga/assembly.py:137-219 (SpatialQuadratureData:
kron_chain collocation matrices, mass = C^T diag(w |det J|) C, stiffness =
sum_ab C_a^T diag(w |det J| (J^-1 J^-T)_ab) C_b) and monoiga/linalg.py:228-262
(FastDiagPreconditioner._separable_weights), in the reference's algorithmic form
(sparse Kronecker collocation, CSR products).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import numpy as np
import scipy.sparse as sp

from .assembly import Rule, kron_list
from .splines import Space


def read_geometry(path):
    """geometry.py:326-344: (spaces, control points) of a save_geometry text file."""
    with open(path) as fh:
        tok = [ln.split() for ln in fh if ln.strip() and not ln.startswith("#")]
    d = int(tok[0][0])
    deg = [int(v) for v in tok[1][:d]]
    cnt = [int(v) for v in tok[2][:d]]
    spaces = [Space(np.array([float(v) for v in tok[3 + l][:cnt[l]]]), deg[l]) for l in range(d)]
    n = int(np.prod([s.dimension for s in spaces]))
    ctrl = np.array([[float(v) for v in r[:d]] for r in tok[3 + d:3 + d + n]])
    return spaces, ctrl


def grid_data(geo_spaces, ctrl, axes):
    """geometry.py:135-186 (order 1): x and jac[..., c, a] on the tensor grid (C order, dir d first)."""
    d = len(geo_spaces)
    grid = ctrl.reshape(tuple(s.dimension for s in reversed(geo_spaces)) + (d,))
    col = [[s.colloc(ax, o).toarray() for o in (0, 1)] for s, ax in zip(geo_spaces, axes)]

    def tab(orders):
        v = grid
        for l in range(d):
            ax = d - 1 - l
            v = np.moveaxis(np.tensordot(col[l][orders[l]], v, axes=(1, ax)), 0, ax)
        return v

    x = tab([0] * d)
    jac = np.empty(x.shape[:-1] + (d, d))
    for a in range(d):
        o = [0] * d
        o[a] = 1
        jac[..., a] = tab(o)
    return x, jac


class QuadData:
    """assembly.py:137-219 on the solution spaces (q = p+1 Gauss per element)."""

    def __init__(self, spaces, geo_spaces, ctrl, fibre=None):
        """``fibre = (sigma_l, sigma_t, direction)``: the transversely isotropic conductivity of BASELINE
        cfg 5 (an extension: the reference's D is a scalar), D = sigma_t I + (sigma_l - sigma_t) f f^T
        with f the unit tangent of map direction ``direction``; the stiffness metric is J^-1 D J^-T."""
        d = len(spaces)
        self.spaces = spaces
        self.rules = [Rule.on(s) for s in spaces]
        self.c0 = [s.colloc(r.points, 0) for s, r in zip(spaces, self.rules)]
        self.c1 = [s.colloc(r.points, 1) for s, r in zip(spaces, self.rules)]
        w = np.ones(())
        for l in reversed(range(d)):
            w = np.multiply.outer(w, self.rules[l].weights)
        self.wgrid = w
        self.x, jac = grid_data(geo_spaces, ctrl, [r.points for r in self.rules])
        self.detj = np.linalg.det(jac)
        self.jinv = np.linalg.inv(jac)
        self.G = None
        if fibre is not None:
            sl, st_, k = fibre
            f = jac[..., :, k] / np.linalg.norm(jac[..., :, k], axis=-1, keepdims=True)
            D = st_ * np.eye(d) + (sl - st_) * f[..., :, None] * f[..., None, :]
            self.G = self.jinv @ D @ np.swapaxes(self.jinv, -1, -2)

    def _ckron(self, deriv=None):
        d = len(self.spaces)
        return kron_list([self.c1[l] if l == deriv else self.c0[l] for l in reversed(range(d))])

    def metric(self, a, b):
        if self.G is not None:
            return self.G[..., a, b]
        return np.einsum("...k,...k->...", self.jinv[..., a, :], self.jinv[..., b, :])

    def mass(self):
        C = self._ckron()
        return sp.csr_matrix(C.T @ sp.diags((self.wgrid * np.abs(self.detj)).ravel()) @ C)

    def stiffness(self):
        d = len(self.spaces)
        base = self.wgrid * np.abs(self.detj)
        K = None
        for a in range(d):
            for b in range(d):
                t = self._ckron(a).T @ sp.diags((base * self.metric(a, b)).ravel()) @ self._ckron(b)
                K = t if K is None else K + t
        return sp.csr_matrix(K)

    def separable_weights(self):
        """linalg.py:228-262."""
        d = len(self.spaces)
        detj = np.abs(self.detj)
        lg = np.log(detj)
        grand = lg.mean()
        mass = [np.exp((lg.mean(axis=tuple(x for x in range(d) if x != d - 1 - l)) if d > 1 else lg)
                       - grand + grand / d) for l in range(d)]
        stiff = []
        for l in range(d):
            coeff = detj * self.metric(l, l)
            den = np.ones_like(coeff)
            for m in range(d):
                if m != l:
                    shp = [1] * d
                    shp[d - 1 - m] = mass[m].size
                    den = den * mass[m].reshape(shp)
            r = coeff / den
            stiff.append(r.mean(axis=tuple(x for x in range(d) if x != d - 1 - l)) if d > 1 else r)
        return mass, stiff
