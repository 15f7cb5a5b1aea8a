"""Quadrature, 1D Gram factors, the Kronecker operator and the reaction mass.

Oracle restatement of monoiga/assembly.py and monoiga/tensorops.py.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import numpy as np
import scipy.sparse as sp


def gauss(q):
    """assembly.py:33-37: Gauss-Legendre nodes/weights on [-1, 1]."""
    return np.polynomial.legendre.leggauss(q)


class Rule:
    """assembly.py:41-82: per-cell Gauss rule over a partition of [0, 1]."""

    def __init__(self, cells, q):
        self.cells = np.asarray(cells, dtype=float)
        self.q = int(q)
        x, w = gauss(self.q)
        lo, hi = self.cells[:-1, None], self.cells[1:, None]
        h = 0.5 * (hi - lo)
        self.nodes = lo + h * (x[None, :] + 1.0)
        self.wts = h * w[None, :]

    @classmethod
    def on(cls, space, q=None, extra=None):
        cells = space.breakpoints
        if extra is not None:
            e = np.asarray(extra, dtype=float)
            cells = np.unique(np.concatenate([cells, e[(e > 0.0) & (e < 1.0)]]))
        return cls(cells, space.degree + 1 if q is None else q)

    @property
    def points(self):
        return self.nodes.ravel()

    @property
    def weights(self):
        return self.wts.ravel()

    @property
    def num_cells(self):
        return self.cells.size - 1


def gram(space, a=0, b=0, weight=None, rule=None):
    """assembly.py:85-101: int w * b_j^(b) * b_i^(a); row = test index."""
    rule = Rule.on(space) if rule is None else rule
    w = rule.weights.copy()
    if weight is not None:
        w = w * np.asarray(weight(rule.points) if callable(weight) else weight).ravel()
    Ci = space.colloc(rule.points, a)
    Cj = space.colloc(rule.points, b)
    return sp.csr_matrix(Ci.T @ sp.diags(w) @ Cj)


def mass_stiff_adv(space, weight=None, rule=None):
    """assembly.py:104-118: (M, K, W), q=p+1 unweighted / p+2 weighted."""
    if rule is None:
        rule = Rule.on(space, space.degree + 1 if weight is None else space.degree + 2)
    return (gram(space, 0, 0, weight, rule), gram(space, 1, 1, weight, rule),
            gram(space, 0, 1, weight, rule))


def time_factors(st, T):
    """assembly.py:125-134: W_t = W[1:,1:], M_t = T * M[1:,1:]."""
    M, _, W = mass_stiff_adv(st.time)
    return sp.csr_matrix(W[1:, 1:]), sp.csr_matrix(T * M[1:, 1:])


def kron_list(mats):
    """tensorops.py:37-42: first factor slowest."""
    out = mats[0]
    for m in mats[1:]:
        out = sp.kron(out, m, format="csr")
    return sp.csr_matrix(out)


def box_spatial(spaces, lengths=None, diffusion=None):
    """assembly.py:222-238 (axis-aligned box): M_s and K_s as Kronecker CSR.

    ``diffusion`` (one value per direction) generalises the scalar D to the
    diagonal conductivity of BASELINE cfg 3: the returned
    stiffness is then sum_a sigma_a K_a-term, and with ``diffusion=None`` the
    plain reference K_s (unit coefficients) is returned.
    """
    d = len(spaces)
    L = np.ones(d) if lengths is None else np.asarray(lengths, float)
    mats = [mass_stiff_adv(s) for s in spaces]
    M = kron_list([L[l] * mats[l][0] for l in reversed(range(d))])
    K = None
    for a in range(d):
        fac = [(mats[l][1] / L[l]) if l == a else (L[l] * mats[l][0])
               for l in reversed(range(d))]
        term = kron_list(fac)
        if diffusion is not None:
            term = diffusion[a] * term
        K = term if K is None else K + term
    return sp.csr_matrix(M), sp.csr_matrix(K)


def mode_product(mat, X, axis):
    """tensorops.py:13-26: out[..i..] = sum_j mat[i, j] X[..j..]."""
    t = np.moveaxis(X, axis, 0)
    out = np.asarray(mat @ t.reshape(t.shape[0], -1)).reshape((mat.shape[0],) + t.shape[1:])
    return np.moveaxis(out, 0, axis)


def two_factor(T, S, x, nt, ns):
    """tensorops.py:45-56: (T kron S) x via T X then (S Y^T)^T."""
    Y = np.asarray(T @ x.reshape(nt, ns)) if T is not None else x.reshape(nt, ns)
    if S is not None:
        Y = np.asarray(S @ Y.T).T
    return Y.reshape(-1)


class KronOp:
    """assembly.py:401-460: sum_k c_k (T_k kron S_k) + optional correction."""

    def __init__(self, nt, ns, terms=(), correction=None):
        self.nt, self.ns = int(nt), int(ns)
        self.terms = [(float(c), T, S) for c, T, S in terms]
        self.correction = correction

    @property
    def shape(self):
        n = self.nt * self.ns
        return (n, n)

    def matvec(self, x):
        x = np.asarray(x, dtype=float).ravel()
        if x.size != self.shape[0]:
            raise ValueError("dimension mismatch: operator of size %d applied to "
                             "vector of size %d" % (self.shape[0], x.size))
        y = np.zeros_like(x)
        for c, T, S in self.terms:
            y += c * two_factor(T, S, x, self.nt, self.ns)
        if self.correction is not None:
            y += self.correction @ x
        return y

    def tosparse(self):
        acc = sp.csr_matrix(self.shape)
        for c, T, S in self.terms:
            acc = acc + c * sp.kron(T, S, format="csr")
        if self.correction is not None:
            acc = acc + sp.csr_matrix(self.correction)
        return sp.csr_matrix(acc)


def spatial_colloc(spaces, q=None, extra=None):
    """assembly.py:137-160: per-direction rules + collocation (dir 1 first)."""
    rules = [Rule.on(s, q, None if extra is None else extra[l]) for l, s in enumerate(spaces)]
    return rules, [s.colloc(r.points, 0) for s, r in zip(spaces, rules)]


def weight_grid(rules, lengths=None):
    """assembly.py:158-166 + |det J| for a box: weights in C order (dir d first)."""
    d = len(rules)
    L = np.ones(d) if lengths is None else np.asarray(lengths, float)
    g = np.asarray(rules[d - 1].weights * L[d - 1])
    for l in reversed(range(d - 1)):
        g = np.multiply.outer(g, rules[l].weights * L[l])
    return g


def field_on_grid(st, coeffs, tcol, scols):
    """assembly.py:272-284."""
    d = st.d
    U = np.asarray(coeffs, dtype=float).reshape(st.coeff_shape)
    out = mode_product(tcol, U, 0)
    for l in range(d):
        out = mode_product(scols[l], out, 1 + (d - 1 - l))
    return out


def reaction_mass(st, T, consts, u, w, lengths=None):
    """assembly.py:287-347: M_R = int int C_r B_i B_j, C_r at q=p+1 Gauss points.

    C_r = c1 (u - a)(u - 1) + c2 w (assembly.py:319).  Assembled as CSR.
    """
    c1, a, c2 = consts["c1"], consts["a"], consts["c2"]
    u = np.asarray(u, float)
    w = np.asarray(w, float)
    if u.size != st.num_dof or w.size != st.num_dof:
        raise ValueError("iterate coefficient vectors must have length N_dof")
    rules, scols = spatial_colloc(st.spatial)
    trule = Rule.on(st.time)
    tcol = st.time_colloc(trule.points, 0)
    tw = trule.weights * T
    uq = field_on_grid(st, u, tcol, scols)
    wq = field_on_grid(st, w, tcol, scols)
    cr = c1 * (uq - a) * (uq - 1.0) + c2 * wq
    ws = weight_grid(rules, lengths).ravel()
    C = kron_list([scols[l] for l in reversed(range(st.d))])
    CT = sp.csc_matrix(C.T)
    ct = tcol.toarray()
    nt, pt = st.num_time, st.time.degree
    slabs = [sp.csr_matrix(CT @ sp.diags(ws * cr[q].ravel()) @ C) for q in range(ct.shape[0])]
    blocks = [[None] * nt for _ in range(nt)]
    for i in range(nt):
        for j in range(max(0, i - pt), min(nt, i + pt + 1)):
            qs = np.nonzero(ct[:, i] * ct[:, j])[0]
            acc = None
            for q in qs:
                term = (ct[q, i] * ct[q, j] * tw[q]) * slabs[q]
                acc = term if acc is None else acc + term
            blocks[i][j] = acc
    return sp.csr_matrix(sp.bmat(blocks, format="csr"))


def reaction_matvec(st, T, consts, u, w, x, lengths=None):
    """Matrix-free M_R x with the same q=p+1 rule (for sizes where CSR is too big).

    Mathematically identical to ``reaction_mass(...) @ x``: interpolate x, u, w
    to the Gauss grid, weight by C_r * w_t * w_s, project back.
    """
    c1, a, c2 = consts["c1"], consts["a"], consts["c2"]
    rules, scols = spatial_colloc(st.spatial)
    trule = Rule.on(st.time)
    tcol = st.time_colloc(trule.points, 0)
    uq = field_on_grid(st, u, tcol, scols)
    wq = field_on_grid(st, w, tcol, scols)
    xq = field_on_grid(st, x, tcol, scols)
    cr = c1 * (uq - a) * (uq - 1.0) + c2 * wq
    wt = trule.weights * T
    ws = weight_grid(rules, lengths)
    g = cr * xq * ws[None] * wt.reshape((-1,) + (1,) * st.d)
    d = st.d
    out = mode_product(tcol.T, g, 0)
    for l in range(d):
        out = mode_product(scols[l].T, out, 1 + (d - 1 - l))
    return out.ravel()
