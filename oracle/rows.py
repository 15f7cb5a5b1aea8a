"""Sampled rows of the reaction mass and of the Spline Upwind terms, for sizes the CSR cannot reach.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference assembles ``M_R`` (assembly.py:287-347) and the SU spatial matrices ``S^s_r``
(stabilization.py:448-489) as global CSR matrices; at BASELINE cfgs 3-4 that is 10^10-10^11 nonzeros.
Row ``i`` of either product only needs the quadrature over the support of the row's basis function,
so these functions evaluate exactly the reference's integrals -- same rules, same weights, same
integrands -- restricted to that support:

* ``reaction_rows``: (M_R x)[i] = sum over the q = p+1 Gauss points of the support elements of
  w_t w_s C_r(u, w) x_h B_i with C_r = c1 (u - a)(u - 1) + c2 w (assembly.py:313-326, 319);
* ``su_rows``: (sum_r sum_k C_m s_r S^t_{r,k} (x) S^s_r) x at row i, with S^t_{r,k} exactly as
  stabilization.py:479-485 (p+2 Gauss on time cells split at the Greville abscissae, tau_k, the
  piecewise-linear time profile) and the S^s_r row as the p+2 Greville-split spatial quadrature of
  theta_{s,r} B_i B_j (stabilization.py:469-474, 487-488; theta from the multilinear space profile,
  stabilization.py:372-398).

Both are pinned against the reference's assembled products on the golden fixtures
(tests/test_oracle_golden.py).
"""

import numpy as np
import scipy.sparse as sp

from .assembly import Rule
from .stab import Indicator  # noqa: F401  (re-exported for callers building indicators)


def _support_cells(space, i, rule):
    """Indices of the rule's cells inside the support [knots[i], knots[i+p+1]] of function i."""
    p = space.degree
    lo, hi = space.knots[i], space.knots[i + p + 1]
    mid = 0.5 * (rule.cells[:-1] + rule.cells[1:])
    return np.nonzero((mid > lo) & (mid < hi))[0]


def _local_1d(space, i, rule, offset=0):
    """Local quadrature data of function i: (points, weights, function indices, values, B_i values).

    ``offset`` = 1 for the constrained time space (full function index = constrained index + 1)."""
    cells = _support_cells(space, i + offset, rule)
    pts = rule.nodes[cells].ravel()
    wts = rule.wts[cells].ravel()
    p = space.degree
    fi = i + offset
    funcs = np.arange(max(fi - p, 0), min(fi + p, space.dimension - 1) + 1)
    C = space.colloc(pts, 0).toarray()
    return pts, wts, funcs, C[:, funcs], C[:, fi]


def _gather(vec, shape, idx_lists):
    """Local block vec.reshape(shape)[ix_(idx...)] with out-of-range (dropped) indices as zeros."""
    V = np.asarray(vec, float).reshape(shape)
    safe = [np.clip(ix, 0, n - 1) for ix, n in zip(idx_lists, shape)]
    blk = V[np.ix_(*safe)].copy()
    for ax, ix in enumerate(idx_lists):
        bad = (ix < 0) | (ix >= shape[ax])
        if bad.any():
            sl = [slice(None)] * len(shape)
            sl[ax] = bad
            blk[tuple(sl)] = 0.0
    return blk


def _field(blk, mats):
    """Evaluate a local coefficient block at the local tensor grid: mats[k] maps axis k."""
    out = blk
    for ax, M in enumerate(mats):
        out = np.moveaxis(np.tensordot(M, np.moveaxis(out, ax, 0), axes=(1, 0)), 0, ax)
    return out


def _split(st, row):
    """Row -> (i_t, [i_1, ..., i_d]) (direction 1 fastest)."""
    ns = st.num_space
    it, rem = divmod(int(row), ns)
    idx = []
    for s in st.spatial:
        rem, k = divmod(rem, s.dimension)
        idx.append(k)
    return it, idx


def reaction_rows(st, T, consts, u, w, x, rows, lengths=None):
    """(M_R x)[rows] with the q = p+1 Gauss rule of assembly.py:313-326 (see module docstring)."""
    c1, a, c2 = consts["c1"], consts["a"], consts["c2"]
    d = st.d
    L = np.ones(d) if lengths is None else np.asarray(lengths, float)
    trule = Rule.on(st.time)
    srules = [Rule.on(s) for s in st.spatial]
    shape = st.coeff_shape
    out = np.empty(len(rows))
    for m, row in enumerate(rows):
        it, isp = _split(st, row)
        tp, tw, tf, Ct, Bt = _local_1d(st.time, it, trule, offset=1)
        loc = [_local_1d(s, isp[l], srules[l]) for l, s in enumerate(st.spatial)]
        idx = [tf - 1] + [loc[l][2] for l in reversed(range(d))]
        mats = [Ct] + [loc[l][3] for l in reversed(range(d))]
        uq = _field(_gather(u, shape, idx), mats)
        wq = _field(_gather(w, shape, idx), mats)
        xq = _field(_gather(x, shape, idx), mats)
        cr = c1 * (uq - a) * (uq - 1.0) + c2 * wq
        wgt = np.multiply.outer(T * tw * Bt, np.ones(1)).ravel()
        for l in reversed(range(d)):
            wgt = np.multiply.outer(wgt, L[l] * loc[l][1] * loc[l][4])
        out[m] = np.sum(wgt * cr * xq)
    return out


def su_time_factors(st, tau, lr):
    """Per rank r: sum_k S^t_{r,k} (N_t x N_t CSR), stabilization.py:463-467, 479-485."""
    p = st.time.degree
    tr = Rule.on(st.time, p + 2, lr.indicator.time_greville)
    tx, tw = tr.points, tr.weights
    out = []
    for r in range(lr.rank):
        prof = lr.time_profile(r, tx)
        acc = None
        for k in range(1, p + 1):
            Ck = st.time_colloc(tx, k)
            Stk = sp.csr_matrix(Ck.T @ sp.diags(tw * tau.evaluate(k, tx) * prof) @ Ck)
            acc = Stk if acc is None else acc + Stk
        out.append(acc)
    return out


def su_rows(st, tau, lr, capacitance, x, rows, lengths=None):
    """(sum_r sum_k C_m s_r S^t_{r,k} (x) S^s_r) x at ``rows`` (see module docstring)."""
    d = st.d
    L = np.ones(d) if lengths is None else np.asarray(lengths, float)
    nt, ns = st.num_time, st.num_space
    X = np.asarray(x, float).reshape(nt, ns)
    if lr.rank == 0:
        return np.zeros(len(rows))
    Ts = su_time_factors(st, tau, lr)
    qs = max(s.degree for s in st.spatial) + 2
    srules = [Rule.on(s, qs, lr.indicator.spatial_grevilles[l]) for l, s in enumerate(st.spatial)]
    sshape = st.spatial_shape
    out = np.zeros(len(rows))
    for m, row in enumerate(rows):
        it, isp = _split(st, row)
        loc = [_local_1d(s, isp[l], srules[l]) for l, s in enumerate(st.spatial)]
        idx = [loc[l][2] for l in reversed(range(d))]
        mats = [loc[l][3] for l in reversed(range(d))]
        axes = [loc[l][0] for l in range(d)]
        wgt = np.ones(1)
        for l in reversed(range(d)):
            wgt = np.multiply.outer(wgt, L[l] * loc[l][1] * loc[l][4])
        wgt = wgt.reshape(tuple(len(loc[l][0]) for l in reversed(range(d))))
        flat = np.ravel_multi_index(np.ix_(*idx), sshape).ravel()   # local spatial functions
        acc = 0.0
        for r in range(lr.rank):
            trow = Ts[r].getrow(it)
            Z = trow.data @ X[trow.indices][:, flat]   # (S^t_r X)[i_t, local]
            zq = _field(Z.reshape(tuple(len(ix) for ix in idx)), mats)
            theta = lr.space_profile(r, axes)
            acc += capacitance * lr.weights[r] * np.sum(wgt * theta * zq)
        out[m] = acc
    return out


def kron_rows(st, terms, x, rows):
    """(sum_k c_k T_k (x) S_{k,d} (x) ... (x) S_{k,1}) x at ``rows``, for Kronecker terms given by their
    factors: ``terms`` = [(c_k, T_k, [S_{k,1}, ..., S_{k,d}])] with every factor a (sparse) matrix --
    the row form of two_factor_matvec with kron_chain spatial factors (tensorops.py:37-56)."""
    d = st.d
    X = np.asarray(x, float).reshape(st.coeff_shape)
    out = np.zeros(len(rows))
    for m, row in enumerate(rows):
        it, isp = _split(st, row)
        acc = 0.0
        for c, T, S in terms:
            rws = [sp.csr_matrix(T).getrow(it)] + [sp.csr_matrix(S[l]).getrow(isp[l]) for l in reversed(range(d))]
            idx = [r.indices for r in rws]
            blk = X[np.ix_(*idx)]
            for r in rws:                      # contract time, then directions d .. 1
                blk = np.tensordot(r.data, blk, axes=(0, 0))
            acc += c * float(blk)
        out[m] = acc
    return out


def mapped_rows(st, geo_spaces, ctrl, terms, x, rows, fibre=None):
    """Rows of the mapped-geometry operator sum_k c_k T_k (x) S_k with S_k the pulled-back quadrature
    mass ('mass': w |det J| B_i B_j) or stiffness ('stiffness': w |det J| grad B_i . J^-1 G J^-T grad B_j,
    G = I or the fibre tensor) of SpatialQuadratureData (assembly.py:137-219, q = p+1 Gauss), evaluated
    on the support of each row's function only.  ``terms`` = [(c_k, T_k, kind_k)]; ``fibre`` as
    oracle.mapped.QuadData.  The map is evaluated with oracle.mapped.grid_data (geometry.py:135-186)."""
    from .mapped import grid_data
    d = st.d
    X = np.asarray(x, float).reshape(st.num_time, st.num_space)
    rules = [Rule.on(s) for s in st.spatial]
    sshape = st.spatial_shape
    out = np.zeros(len(rows))
    for m, row in enumerate(rows):
        it, isp = _split(st, row)
        loc = [_local_1d(s, isp[l], rules[l]) for l, s in enumerate(st.spatial)]
        idx = [loc[l][2] for l in reversed(range(d))]
        flat = np.ravel_multi_index(np.ix_(*idx), sshape).ravel()
        pts = [loc[l][0] for l in range(d)]
        xg, jac = grid_data(geo_spaces, ctrl, pts)             # (Q_d..Q_1, d), (.., d, d)
        detj = np.abs(np.linalg.det(jac))
        jinv = np.linalg.inv(jac)
        if fibre is not None:
            sl, stv, kdir = fibre
            f = jac[..., :, kdir] / np.linalg.norm(jac[..., :, kdir], axis=-1, keepdims=True)
            Dm = stv * np.eye(d) + (sl - stv) * f[..., :, None] * f[..., None, :]
            metric = jinv @ Dm @ np.swapaxes(jinv, -1, -2)
        else:
            metric = jinv @ np.swapaxes(jinv, -1, -2)
        w = np.ones(())
        for l in reversed(range(d)):
            w = np.multiply.outer(w, loc[l][1])
        w = w * detj
        # B_i and its parametric gradient at the local grid; the trial field and its gradient from the
        # local coefficient block of (T_k X)[i_t]
        bi = [loc[l][4] for l in range(d)]
        dsp = [st.spatial[l].colloc(pts[l], 1).toarray() for l in range(d)]
        dbi = [dsp[l][:, isp[l]] for l in range(d)]
        dmat = [dsp[l][:, loc[l][2]] for l in range(d)]

        def outer(vecs):
            g = np.ones(())
            for l in reversed(range(d)):
                g = np.multiply.outer(g, vecs[l])
            return g

        Bi = outer(bi)
        gBi = [outer([dbi[l] if l == a else bi[l] for l in range(d)]) for a in range(d)]
        acc = 0.0
        for c, T, kind in terms:
            trow = sp.csr_matrix(T).getrow(it)
            Z = (trow.data @ X[trow.indices][:, flat]).reshape(tuple(len(ix) for ix in idx))
            if kind == "mass":
                zq = _field(Z, [loc[l][3] for l in reversed(range(d))])
                acc += c * np.sum(w * Bi * zq)
            else:
                gz = [_field(Z, [(dmat[l] if l == a else loc[l][3]) for l in reversed(range(d))]) for a in range(d)]
                val = 0.0
                for a in range(d):
                    for b in range(d):
                        val = val + np.sum(w * metric[..., a, b] * gBi[a] * gz[b])
                acc += c * val
        out[m] = acc
    return out
