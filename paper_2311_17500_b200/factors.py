"""Host setup of the small factor tables consumed by the CUDA kernels.

* Spline Upwind: upwind weights tau_k (stabilization.py:84-145), truncated SVD
  of the indicator (stabilization.py:401-418), per-rank time bands
  sum_k S^t_{r,k} (stabilization.py:461-486) and the 1D hat-weighted triple
  products that generate the spatial stencils S^s_r on the device
  (stabilization.py:469-488, see ``hat_triple``).
* Fast diagonalisation: spatial eigen-pairs (linalg.py:75-89, 264-307) and
  the bordered time pencil in REAL block form (linalg.py:127-173; see
  ``RealTimePencil``).

All tables are <= O(n^2) with n <= a few hundred.
"""

import numpy as np
import scipy.linalg as sla

from ._blas import single_thread_blas as _single_thread_blas
from .errors import DecompositionError, StabilizationError
from .spaces import (SplineSpace, basis_table, cells_with, gauss_rule, greville,
                     time_factors, to_band, univariate_factors)


# --------------------------------------------------------------------------
# Spline Upwind
# --------------------------------------------------------------------------

class UpwindWeights:
    """tau_k (k = 1..p) as splines of degree p-k on the time breakpoints."""

    def __init__(self, spaces, coeffs, residual):
        self.spaces, self.coeffs, self.residual = spaces, coeffs, residual

    def evaluate(self, k, x):
        return basis_table(self.spaces[k - 1], x, 0) @ self.coeffs[k - 1]


def upwind_weights(tspace):
    """Cached per time space (knots, degree); see _upwind_weights."""
    key = (tuple(np.asarray(tspace.knots, float).tolist()), int(tspace.degree))
    hit = _TAU_CACHE.get(key)
    if hit is None:
        hit = _upwind_weights(tspace)
        _TAU_CACHE[key] = hit
    return hit


_TAU_CACHE = {}


def _upwind_weights(tspace):
    """Solve the orthogonality conditions of stabilization.py:84-145.

    For every near-diagonal pair (i, i+l), l = 1..p, of the full time basis,
    sum_k int tau_k b_j^(k) b_i^(k) = -int b_j' b_i.  The stacked system is
    square; it is solved by least squares after column equilibration (the
    order-k weight scales like h^(1-2k)).
    """
    p = tspace.degree
    bp = tspace.breakpoints
    spaces = []
    for k in range(1, p + 1):
        q = p - k
        knots = np.concatenate([np.zeros(q + 1), bp[1:-1], np.ones(q + 1)])
        spaces.append(SplineSpace(knots, q))
    x, w = gauss_rule(bp, 2 * p)
    B = [basis_table(tspace, x, k) for k in range(p + 1)]
    Phi = [basis_table(s, x, 0) for s in spaces]
    n = tspace.dimension
    rows, rhs = [], []
    for i in range(n - 1):
        for j in range(i + 1, min(i + p, n - 1) + 1):
            rows.append(np.concatenate([(w * B[k][:, i] * B[k][:, j]) @ Phi[k - 1]
                                        for k in range(1, p + 1)]))
            rhs.append(-np.dot(w * B[0][:, i], B[1][:, j]))
    G, b = np.asarray(rows), np.asarray(rhs)
    scale = np.linalg.norm(G, axis=0)
    scale[scale == 0.0] = 1.0
    sol = np.linalg.lstsq(G / scale, b, rcond=None)[0] / scale
    res = np.max(np.abs(G @ sol - b)) / max(np.max(np.abs(b)), 1e-300)
    if res > 1e-8:
        raise StabilizationError("upwind weight conditions not satisfied (residual %.3e)" % res)
    sizes = np.cumsum([0] + [s.dimension for s in spaces])
    return UpwindWeights(spaces, [sol[sizes[k]:sizes[k + 1]] for k in range(p)], res)


class LowRankIndicator:
    """Truncated SVD Theta ~ U_r s_r V_r^T with rank = min{k: tail <= tol ||Theta||}."""

    def __init__(self, values, rank, time_factors, space_factors, weights, tol):
        self.values = values
        self.rank = int(rank)
        self.time_factors = time_factors
        self.space_factors = space_factors
        self.weights = weights
        self.tol = tol


def lowrank_factorize(values, tol):
    """stabilization.py:401-418 (numpy SVD on the host, rank >= 1 unless Theta = 0; large wide
    indicators through the Gram matrix, see below)."""
    if not 0.0 < tol < 1.0:
        raise ValueError("tolerance must lie in (0, 1)")
    is_torch = type(values).__module__.startswith("torch")   # (a tensor's .values is a method)
    th = values if is_torch else getattr(values, "values", values)
    if type(th).__module__.startswith("torch"):
        lr = _lowrank_device(th, tol)
        if lr is not None:
            return lr
        th = th.cpu().numpy()
    th = np.asarray(th, float)
    nrm = np.linalg.norm(th)
    nt, ns = th.shape
    if nrm == 0.0:
        return LowRankIndicator(th, 0, np.zeros((nt, 0)), np.zeros((ns, 0)), np.zeros(0), tol)
    if nt * ns > GRAM_MIN_SIZE and ns >= 8 * nt:
        # wide indicator (N_s >> N_t): eigen-decomposition of the N_t x N_t Gram matrix is ~40x
        # cheaper than the full SVD at cfg 3 (0.1 vs 4 s).  The rank decision uses the same
        # tails (eigenvalues = s^2); when a tail sits within 1e-8 of the cut, the full SVD decides.
        lam, W = np.linalg.eigh(th @ th.T)
        lam, W = np.clip(lam[::-1], 0.0, None), W[:, ::-1]
        tails2 = np.append(np.cumsum(lam[::-1])[::-1], 0.0)
        cut2 = (tol * nrm) ** 2
        if np.min(np.abs(tails2 - cut2)) > 1e-8 * nrm ** 2:
            rank = max(int(np.argmax(tails2 <= cut2)), 1)
            s = np.sqrt(lam[:rank])          # > 0: tails2[rank-1] > cut2 >= tails2[rank]
            V = (th.T @ W[:, :rank]) / s
            return LowRankIndicator(th, rank, np.ascontiguousarray(W[:, :rank]), V, s[:rank].copy(), tol)
    with _single_thread_blas(th.size < 1 << 20):
        U, s, Vt = np.linalg.svd(th, full_matrices=False)
    tails = np.sqrt(np.append(np.cumsum((s ** 2)[::-1])[::-1], 0.0))
    rank = max(int(np.argmax(tails <= tol * nrm)), 1)
    return LowRankIndicator(th, rank, U[:, :rank], Vt[:rank].T.copy(), s[:rank].copy(), tol)


GRAM_MIN_SIZE = 2_000_000





def _lowrank_device(th, tol):
    """The Gram path of lowrank_factorize with the indicator on the device: Theta Theta^T and the
    spatial factors Theta^T W / s by cuBLAS DGEMM, the N_t x N_t eigendecomposition and the rank decision
    on the host.  None when the full SVD must decide (small / not wide / tail at the cut)."""
    import torch
    nt, ns = th.shape
    if not (nt * ns > GRAM_MIN_SIZE and ns >= 8 * nt):
        return None
    nrm = float(torch.linalg.norm(th).item())
    if nrm == 0.0:
        return None
    lam, W = np.linalg.eigh((th @ th.T).cpu().numpy())
    lam, W = np.clip(lam[::-1], 0.0, None), W[:, ::-1]
    tails2 = np.append(np.cumsum(lam[::-1])[::-1], 0.0)
    cut2 = (tol * nrm) ** 2
    if np.min(np.abs(tails2 - cut2)) <= 1e-8 * nrm ** 2:
        return None
    rank = max(int(np.argmax(tails2 <= cut2)), 1)
    s = np.sqrt(lam[:rank])
    Wr = np.ascontiguousarray(W[:, :rank])
    V = (th.T @ torch.from_numpy(Wr).to(th.device)).cpu().numpy() / s
    return LowRankIndicator(th, rank, Wr, V, s[:rank].copy(), tol)


def hat_values(nodes, x):
    """Piecewise-linear nodal basis on ``nodes`` evaluated at x: (len(x), len(nodes)).

    Matches np.interp / linear RegularGridInterpolator after clipping x to
    [nodes[0], nodes[-1]] (stabilization.py:362-398).
    """
    nodes = np.asarray(nodes, float)
    x = np.clip(np.asarray(x, float), nodes[0], nodes[-1])
    H = np.zeros((x.size, nodes.size))
    j = np.clip(np.searchsorted(nodes, x, side="right") - 1, 0, nodes.size - 2)
    t = (x - nodes[j]) / (nodes[j + 1] - nodes[j])
    H[np.arange(x.size), j] = 1.0 - t
    H[np.arange(x.size), j + 1] = t
    return H


def _shifted(A, lo, hi):
    """Column-shifted view helper: S[:, s - lo, i] = A[:, i + s] (0 outside), s in [lo, hi]."""
    nq, n = A.shape
    P = np.zeros((nq, n + hi - lo))
    P[:, -lo:-lo + n] = A
    return [P[:, s - lo:s - lo + n] for s in range(lo, hi + 1)]


def su_time_bands(st, tau, lowrank, capacitance):
    """Per rank r: band of C_m s_r sum_k int tau_k prof_r b_i^(k) b_j^(k) dt.

    Parametric time integrals, p+2 Gauss points on cells split at the
    constrained time Greville abscissae (stabilization.py:461-486).  The
    k-sum is a legal reassociation (one spatial factor per rank,
    stabilization.py:439-445).  Only the 2p+1 diagonals are formed.
    Returns (R, N_t, 2p+1).
    """
    p = st.time.degree
    tg = st.time_greville()
    x, w = gauss_rule(cells_with(st.time, tg), p + 2)
    prof = hat_values(tg, x) @ lowrank.time_factors          # (nq, R)
    nt = st.num_time
    bands = np.zeros((lowrank.rank, nt, 2 * p + 1))
    for k in range(1, p + 1):
        Bk = basis_table(st.time, x, k)[:, 1:]
        tk = tau.evaluate(k, x)
        shifts = _shifted(Bk, -p, p)                          # Bk[:, i + dj - p]
        wk = (w * tk)[:, None] * prof                         # (nq, R)
        for dj in range(2 * p + 1):
            prod = Bk * shifts[dj]                            # (nq, nt): b_i b_{i+dj-p}
            bands[:, :, dj] += wk.T @ prod
    coef = capacitance * lowrank.weights
    return bands * coef[:, None, None]


def su_time_lift(st, tau, lowrank, capacitance):
    """Per rank r: C_m s_r sum_k int tau_k prof_r b_i^(k) b_0^(k) dt for the constrained rows i -- the
    column of the full SU time factor coupling them to the dropped b_0 (u0 lifting).  Same rule as
    su_time_bands.  Returns (R, N_t) (nonzero in the first p rows only)."""
    p = st.time.degree
    tg = st.time_greville()
    x, w = gauss_rule(cells_with(st.time, tg), p + 2)
    prof = hat_values(tg, x) @ lowrank.time_factors          # (nq, R)
    out = np.zeros((lowrank.rank, st.num_time))
    for k in range(1, p + 1):
        Bf = basis_table(st.time, x, k)
        wk = (w * tau.evaluate(k, x))[:, None] * prof         # (nq, R)
        out += wk.T @ (Bf[:, 1:] * Bf[:, :1])
    return out * (capacitance * lowrank.weights)[:, None]


def hat_triple(space, length=1.0):
    """H[i, dj, k] = L * int hat_{i+k-KO}(x) b_i(x) b_{i+dj-p}(x) dx.

    The spatial SU matrix of rank r is the theta_r-weighted mass matrix with
    theta_r multilinear on the Greville grid (stabilization.py:469-488), i.e.
    S^s_r[i, j] = sum_k theta_r[k] prod_l H_l[i_l, j_l - i_l + p, k_l - i_l + KO].
    Computed with p+2 Gauss points on cells split at the Greville abscissae
    (exact: the integrand is a polynomial of degree 2p+1 per cell), band by
    band.  Returns (H, KO) with H of shape (n, 2p+1, 2*KO+1); cached per
    (knots, degree, length) because it depends on the space only.
    """
    key = (tuple(np.asarray(space.knots, float).tolist()), int(space.degree), float(length))
    hit = _HAT_CACHE.get(key)
    if hit is None:
        hit = _hat_triple(space, length)
        _HAT_CACHE[key] = hit
    return hit[0].copy(), hit[1]


_HAT_CACHE = {}


def _hat_triple(space, length):
    p = space.degree
    n = space.dimension
    g = greville(space)
    x, w = gauss_rule(cells_with(space, g), p + 2)
    w = w * length
    B = basis_table(space, x, 0)
    Hat = hat_values(g, x)
    KO = p + 1
    H = np.zeros((n, 2 * p + 1, 2 * KO + 1))
    Bs = _shifted(B, -p, p)
    Hs = _shifted(Hat, -KO, KO)
    WB = w[:, None] * B
    inside = 0.0
    for dj in range(2 * p + 1):
        WBB = WB * Bs[dj]
        for dk in range(2 * KO + 1):
            H[:, dj, dk] = (WBB * Hs[dk]).sum(axis=0)
            inside += (np.abs(WBB) * np.abs(Hs[dk])).sum()
    # every nonzero triple product must fall inside the stored window: the windowed sum of
    # |w b_i b_j hat_k| must equal the unrestricted one, sum_q |w| (sum_i |b|)^2 (sum_k |hat|)
    total = float((np.abs(w) * np.abs(B).sum(axis=1) ** 2 * np.abs(Hat).sum(axis=1)).sum())
    if total - inside > 1e-12 * max(total, 1e-300):
        raise StabilizationError("hat triple-product window too small")
    return H, KO


# --------------------------------------------------------------------------
# Fast diagonalisation
# --------------------------------------------------------------------------

def _centro_eigh(K, M):
    """eigh(K, M) of a centrosymmetric pencil (J K J = K, J M J = M, J the index reversal: uniform
    open knot vectors) as two half-size problems on the even and odd subspaces.  The hs = n - n/2
    symmetric eigenvectors come first, then the h = n/2 skew ones, every pair of mirrored rows
    EXACTLY equal (or opposite): the device then applies U_l^T / U_l as two half-size products
    (csrc/mode_fold.cuh).  Returns None when the pencil is not centrosymmetric to rounding."""
    n = K.shape[0]
    if n < 4:
        return None
    for A in (K, M):
        if np.max(np.abs(A - A[::-1, ::-1])) > 1e-13 * np.max(np.abs(A)):
            return None
    h = n // 2
    hs = n - h
    r = 1.0 / np.sqrt(2.0)
    Ps = np.zeros((n, hs))
    Pa = np.zeros((n, h))
    for k in range(h):
        Ps[k, k] = Ps[n - 1 - k, k] = r
        Pa[k, k], Pa[n - 1 - k, k] = r, -r
    if n % 2:
        Ps[h, h] = 1.0
    out_l, out_v = [], []
    for P in (Ps, Pa):
        Kb, Mb = P.T @ K @ P, P.T @ M @ P
        lam, V = sla.eigh(0.5 * (Kb + Kb.T), 0.5 * (Mb + Mb.T))
        out_l.append(lam)
        out_v.append(V)
    U = np.zeros((n, n))
    top = out_v[0][:h] * r
    U[:h, :hs] = top
    U[n - 1 - np.arange(h), :hs] = top
    if n % 2:
        U[h, :hs] = out_v[0][h]
    top = out_v[1] * r
    U[:h, hs:] = top
    U[n - 1 - np.arange(h), hs:] = -top
    return np.concatenate(out_l), U


def spatial_eigs(st, lengths=None):
    """eigh(K_l, M_l) per direction with the box separable weights.

    The solver always passes spatial quadrature data (solver.py:193-202),
    so the weighted factors of linalg.py:290-300 are used; on a box with
    side lengths L they are mass weight det^(1/d) and stiffness weight
    det^(1/d)/L_l^2 (linalg.py:228-262), i.e. exactly 1 on the unit box.
    """
    d = st.num_spatial_dims
    L = np.ones(d) if lengths is None else np.asarray(lengths, float)
    cm = np.prod(L) ** (1.0 / d)
    out = []
    for l, s in enumerate(st.spatial):
        M, K, _ = univariate_factors(s)
        Kl, Ml = (cm / L[l] ** 2) * K, cm * M
        try:
            with _single_thread_blas():
                split = _centro_eigh(Kl, Ml)
                lam, U = split if split is not None else sla.eigh(Kl, Ml)
        except sla.LinAlgError as exc:
            raise DecompositionError("generalized eigendecomposition failed: %s" % exc) from exc
        out.append((U, lam))
    return out


def mapped_spatial_eigs(sd):
    """linalg.py:286-297 on a mapped geometry: eigh(K_l, M_l) of the univariate factors weighted by
    the separable surrogates of the pulled-back measures (geometry.separable_weights), on the
    q = p+1 Gauss rule of the mesh (the rule of SpatialQuadratureData)."""
    from .geometry import separable_weights
    from .spaces import gram
    w_mass, w_stiff = separable_weights(sd)
    out = []
    for l, s in enumerate(sd.spaces):
        x, w = sd.rules[l]
        M = gram(s, 0, 0, x, w * w_mass[l])
        K = gram(s, 1, 1, x, w * w_stiff[l])
        try:
            lam, U = sla.eigh(K, M)
        except sla.LinAlgError as exc:
            raise DecompositionError("generalized eigendecomposition failed: %s" % exc) from exc
        out.append((U, lam))
    return out


class RealTimePencil:
    """Bordered time pencil in real 2x2-block form.

    The reference (linalg.py:127-173) whitens the interior advection block
    with the Cholesky factor of the interior mass, diagonalises the skew
    matrix S over C (purely imaginary eigenvalues in conjugate pairs) and
    borders the basis with the mass-orthogonal complement column [t; rho].
    Here the same whitened S is put in REAL Schur form S = Z T Z^T
    (T block diagonal with 2x2 skew blocks for a normal matrix), so

        Q^T M_t Q = I,   Q^T W_t Q = [[T, g], [-g^T, sigma]]

    with Q = [[L^-T Z, t], [0, rho]] real.  The surrogate inverse is basis
    independent, so P^-1 is identical to the complex form; the apply runs in
    real arithmetic at half the flops and its result is real by
    construction (the reference's imaginary-residue check, linalg.py:347-352,
    has nothing to test; the pencil quality is checked here instead).
    """

    def __init__(self, Wt, Mt, cond_limit=1e12):
        W = np.asarray(Wt, float)
        M = np.asarray(Mt, float)
        n = W.shape[0]
        if n < 2:
            raise ValueError("temporal dimension must be at least 2")
        Wi, Mi, wb, mb = W[:-1, :-1], M[:-1, :-1], W[:-1, -1], M[:-1, -1]
        try:
            L = np.linalg.cholesky(Mi)
        except np.linalg.LinAlgError as exc:
            raise DecompositionError("temporal mass block not SPD: %s" % exc) from exc
        S = sla.solve_triangular(L, sla.solve_triangular(L, Wi, lower=True).T, lower=True).T
        S = 0.5 * (S - S.T)
        T, Z = sla.schur(S, output="real")
        Ui = sla.solve_triangular(L.T, Z, lower=False)
        v = sla.cho_solve((L, True), -mb)
        s2 = float(v @ Mi @ v + 2.0 * (v @ mb) + M[-1, -1])
        if s2 <= 0:
            raise DecompositionError("temporal mass matrix not positive definite")
        t, rho = v / np.sqrt(s2), 1.0 / np.sqrt(s2)
        Q = np.zeros((n, n))
        Q[:-1, :-1] = Ui
        Q[:-1, -1] = t
        Q[-1, -1] = rho
        with _single_thread_blas(True):
            condq = np.linalg.cond(Q)
        if condq > cond_limit:
            raise DecompositionError("temporal pencil eigenvectors ill-conditioned")
        # 2x2 block partition of the quasi-triangular T (skew => block diagonal)
        m = n - 1
        blocks = []
        i = 0
        while i < m:
            if i + 1 < m and T[i + 1, i] != 0.0:
                blocks.append((i, 2))
                i += 2
            else:
                blocks.append((i, 1))
                i += 1
        Tb = np.zeros_like(T)
        for i0, sz in blocks:
            Tb[i0:i0 + sz, i0:i0 + sz] = T[i0:i0 + sz, i0:i0 + sz]
        Delta = Q.T @ W @ Q
        resid = Delta.copy()
        resid[:-1, :-1] -= Tb
        resid[:-1, -1] = 0.0
        resid[-1, :] = 0.0
        scale = max(np.max(np.abs(Delta)), 1e-300)
        if np.max(np.abs(resid)) > 1e-8 * scale:
            raise DecompositionError("time pencil is not block-arrowhead (residue %.3e)"
                                     % (np.max(np.abs(resid)) / scale))
        self.Q = Q
        self.blocks = blocks
        self.T = Tb
        self.g = Delta[:-1, -1].copy()          # upper border (lower = -g^T)
        self.g_low = Delta[-1, :-1].copy()
        self.sigma = float(Delta[-1, -1])
        self.n = n

    def coupling(self):
        """(a, b, c, e) per interior index: 2x2 block [[a, b], [c, e]] data.

        Returned as four length-(n-1) arrays describing, for each interior
        row i, its block partner: for a 1x1 block b = c = 0 and the partner is
        itself.  ``partner[i]`` gives the other row of the block.
        """
        m = self.n - 1
        diag = np.zeros(m)
        off = np.zeros(m)
        partner = np.arange(m)
        for i0, sz in self.blocks:
            if sz == 1:
                diag[i0] = self.T[i0, i0]
            else:
                diag[i0] = self.T[i0, i0]
                diag[i0 + 1] = self.T[i0 + 1, i0 + 1]
                off[i0] = self.T[i0, i0 + 1]
                off[i0 + 1] = self.T[i0 + 1, i0]
                partner[i0], partner[i0 + 1] = i0 + 1, i0
        return diag, off, partner


def time_pencil(st, final_time):
    Wt, Mt = time_factors(st, final_time)
    with _single_thread_blas():
        return RealTimePencil(Wt, Mt)
