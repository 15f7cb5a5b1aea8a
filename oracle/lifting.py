"""Oracle EXTENSION: the relaxed fixed-point solve with nonzero initial data (u0 lifting).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference cannot take u0 != 0: its trial space drops the first time function (bspline.py:384-387)
and every field evaluation pads that slab with zeros (``_full_time_tensor``, fields.py:8-12), so only
source terms drive its solutions.  BASELINE's stimuli are initial data, so the
build adds the standard lifting; this module is its CPU restatement, built from the oracle's
reference restatements (pinned against the reference in tests/test_oracle_golden.py) and itself
pinned at u0 = 0 against the reference's own ``fixed_point_solve`` fixtures.

Specification of the lifted problem:

* u_h(x, t) = u0_h(x) b_0(t) + sum_i u~_i B_i(x, t) with u~ in the reference's trial space and
  u0_h = sum_s u0(gamma_s) B_s(x) the Schoenberg quasi-interpolant at the spatial Greville abscissae
  (monotone: a step u0 stays in [0, 1]).  w0 = 0 (no lifting of w).
* Sweep k solves, for every constrained test function, a_k(u~, v) = F(v) - a_k(u0_h b_0, v), where
  a_k is the reference's bilinear form of the sweep (solver.py:213-236): C_m W (x) M_s, D M (x) K_s,
  the reaction and the Spline Upwind terms, each with the full time factor's column 0 for the lifted
  part.  The reaction is M_R at C_r(u^k_h, w^k_h) with the LIFTED iterate; the Kronecker a c1 term
  is used iff that lifted iterate and w vanish identically (with u0 = 0 exactly the reference's test).
* The indicator is compute_theta (stabilization.py:235-339) of the lifted field (the dropped slab
  padded with u0 instead of zeros), on the reference's constrained Greville grid with its windows.
* The recovery right-hand side is g = b (M (x) M_s) u_h over the full time factor (column 0 included).

With u0 = 0 every formula reduces to the reference's.
"""

import warnings

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import assembly as asm
from . import krylov
from . import stab as ostab
from .fastdiag import FastDiag
from .splines import make_space_time  # noqa: F401  (callers build spaces with it)


def greville_lift(spaces, u0):
    """Quasi-interpolant coefficients of u0 (callable on (n, d) points, or given coefficients), C order."""
    if not callable(u0):
        return np.asarray(u0, float).ravel()
    g = [s.greville() for s in spaces]
    d = len(spaces)
    mesh = np.meshgrid(*[g[l] for l in reversed(range(d))], indexing="ij")
    pts = np.stack([mesh[d - 1 - l].ravel() for l in range(d)], axis=1)
    return np.asarray(u0(pts), float).ravel()


def full_time_factors(st, T):
    """Full (n_t x n_t) W and T M (assembly.py:104-118, 125-134 before dropping row/column 0)."""
    M, _, W = asm.mass_stiff_adv(st.time)
    return sp.csr_matrix(W), sp.csr_matrix(T * M)


def full_coeffs(st, uc, u0):
    """(n_t, n_d, ..., n_1) tensor: slab 0 = u0 (zeros without lifting), the rest = the iterate."""
    full = np.zeros((st.time.dimension,) + st.spatial_shape)
    full[1:] = np.asarray(uc, float).reshape(st.coeff_shape)
    if u0 is not None:
        full[0] = np.asarray(u0, float).reshape(st.spatial_shape)
    return full


def field(st, full, tcol, scols):
    """field_on_grid (assembly.py:272-284) with a FULL time collocation."""
    out = asm.mode_product(tcol, full, 0)
    for l in range(st.d):
        out = asm.mode_product(scols[l], out, 1 + (st.d - 1 - l))
    return out


def reaction_mass_full(st, T, consts, u_full, w_full, lengths=None):
    """assembly.py:287-347 with the full time basis on both sides: an (n_t N_s) x (n_t N_s) CSR whose
    [1:, 1:] block is the reference's M_R and whose [1:, 0] block couples the lifted slab."""
    c1, a, c2 = consts["c1"], consts["a"], consts["c2"]
    rules, scols = asm.spatial_colloc(st.spatial)
    trule = asm.Rule.on(st.time)
    tcol = st.time.colloc(trule.points, 0)
    tw = trule.weights * T
    uq = field(st, u_full, tcol, scols)
    wq = field(st, w_full, tcol, scols)
    cr = c1 * (uq - a) * (uq - 1.0) + c2 * wq
    ws = asm.weight_grid(rules, lengths).ravel()
    C = asm.kron_list([scols[l] for l in reversed(range(st.d))])
    CT = sp.csc_matrix(C.T)
    ct = tcol.toarray()
    n = st.time.dimension
    pt = st.time.degree
    slabs = [sp.csr_matrix(CT @ sp.diags(ws * cr[q].ravel()) @ C) for q in range(ct.shape[0])]
    blocks = [[None] * n for _ in range(n)]
    for i in range(n):
        for j in range(max(0, i - pt), min(n, i + pt + 1)):
            acc = None
            for q in np.nonzero(ct[:, i] * ct[:, j])[0]:
                term = (ct[q, i] * ct[q, j] * tw[q]) * slabs[q]
                acc = term if acc is None else acc + term
            blocks[i][j] = acc
    return sp.csr_matrix(sp.bmat(blocks, format="csr"))


def su_full_terms(tau, lr, st, cm, lengths=None):
    """assemble_stabilization (stabilization.py:448-489) with the FULL time collocation: the same
    (coef, S^t_{r,k}, S^s_r) terms with S^t of size n_t x n_t (row/column 0 = the dropped function)."""
    p = st.time.degree
    if lr.rank == 0:
        return []
    tr = asm.Rule.on(st.time, p + 2, lr.indicator.time_greville)
    tx, tw = tr.points, tr.weights
    qs = max(s.degree for s in st.spatial) + 2
    rules, scols = asm.spatial_colloc(st.spatial, qs, lr.indicator.spatial_grevilles)
    C = asm.kron_list([scols[l] for l in reversed(range(st.d))])
    wg = asm.weight_grid(rules, lengths)
    axes = [r.points for r in rules]
    out = []
    for r in range(lr.rank):
        prof = lr.time_profile(r, tx)
        Ss = sp.csr_matrix(C.T @ sp.diags((wg * lr.space_profile(r, axes)).ravel()) @ C)
        for k in range(1, p + 1):
            Ck = st.time.colloc(tx, k)
            St = sp.csr_matrix(Ck.T @ sp.diags(tw * tau.evaluate(k, tx) * prof) @ Ck)
            out.append((cm * lr.weights[r], St, Ss))
    return out


def compute_theta(st, T, cm, D, consts, source, uc, wc, u0=None, lengths=None):
    """stabilization.py:235-339 on a box (diagonal map: jinv = 1/L, no Hessian) for the lifted field.

    ``D`` is the reference's scalar or one value per direction (the anisotropic extension).
    Returns the N_t x N_s indicator values."""
    d = st.d
    L = np.ones(d) if lengths is None else np.asarray(lengths, float)
    Dv = np.atleast_1d(np.asarray(D, float))
    Dv = np.repeat(Dv, d) if Dv.size == 1 else Dv
    c1, a, c2 = consts["c1"], consts["a"], consts["c2"]
    trule = asm.Rule.on(st.time)
    srules = [asm.Rule.on(s) for s in st.spatial]
    tc = [st.time.colloc(trule.points, o) for o in (0, 1)]
    sc = [[s.colloc(r.points, o) for o in range(3)] for s, r in zip(st.spatial, srules)]
    U = full_coeffs(st, uc, u0)
    Wf = full_coeffs(st, wc, None)

    def fld(X, orders, torder):
        return field(st, X, tc[torder], [sc[l][orders[l]] for l in range(d)])

    u_val = fld(U, [0] * d, 0)
    u_dtau = fld(U, [0] * d, 1)
    w_val = fld(Wf, [0] * d, 0)
    lap = np.zeros_like(u_val)
    for ax in range(d):
        o = [0] * d
        o[ax] = 2
        lap += Dv[ax] * fld(U, o, 0) / L[ax] ** 2
    res = cm * (u_dtau / T) - lap + c1 * u_val * (u_val - a) * (u_val - 1.0) + c2 * u_val * w_val
    if source is not None:
        mesh = np.meshgrid(*[srules[l].points * L[l] for l in reversed(range(d))], indexing="ij")
        xs = np.stack([mesh[d - 1 - l].ravel() for l in range(d)], axis=1)
        qs = xs.shape[0]
        fv = np.empty((trule.points.size, qs))
        for i, t in enumerate(trule.points * T):
            fv[i] = np.asarray(source(xs, np.full(qs, t)), float).reshape(qs)
        res = res - fv.reshape(res.shape)
    absres = np.abs(res)
    denom = cm * (np.max(np.abs(u_val), initial=0.0) / T + np.max(np.abs(u_dtau), initial=0.0) / T)
    shape = [trule.num_cells, trule.q]
    for l in reversed(range(d)):
        shape += [srules[l].num_cells, srules[l].q]
    emax = absres.reshape(shape)
    for ax in reversed(range(1, 2 * (d + 1), 2)):
        emax = emax.max(axis=ax)
    # windows exactly as stabilization.py:318-326: constrained row c takes window_elements(c) of the
    # full time space
    out = np.stack([emax[a_:b_].max(axis=0) for a_, b_ in (st.time.window_elements(c) for c in range(st.num_time))])
    for l in reversed(range(d)):
        axis = 1 + (d - 1 - l)
        wins = [st.spatial[l].window_elements(i) for i in range(st.spatial[l].dimension)]
        moved = np.moveaxis(out, axis, 0)
        moved = np.stack([moved[a_:b_].max(axis=0) for a_, b_ in wins], axis=0)
        out = np.moveaxis(moved, 0, axis)
    numer = out.reshape(st.num_time, st.num_space)
    if denom > 0.0:
        return np.minimum(numer / denom, 1.0)
    theta = np.zeros_like(numer)
    hot = numer > 1e-12 * numer.max(initial=0.0)
    if np.any(hot) and numer.max(initial=0.0) > 0.0:
        warnings.warn("residual indicator denominator vanished with a nonzero residual", RuntimeWarning)
        theta[hot] = 1.0
    return theta


def load_vector(st, T, source, lengths=None):
    """rhs_vectors f (assembly.py:350-398) on a box."""
    if source is None:
        return np.zeros(st.num_dof)
    d = st.d
    L = np.ones(d) if lengths is None else np.asarray(lengths, float)
    rules, scols = asm.spatial_colloc(st.spatial)
    trule = asm.Rule.on(st.time)
    mesh = np.meshgrid(*[rules[l].points * L[l] for l in reversed(range(d))], indexing="ij")
    xs = np.stack([mesh[d - 1 - l].ravel() for l in range(d)], axis=1)
    qs = xs.shape[0]
    fv = np.empty((trule.points.size, qs))
    for i, t in enumerate(trule.points * T):
        fv[i] = np.asarray(source(xs, np.full(qs, t)), float).reshape(qs)
    ws = asm.weight_grid(rules, lengths).ravel()
    vals = fv * ws[None, :] * (trule.weights * T)[:, None]
    tcol = st.time_colloc(trule.points, 0)
    C = asm.kron_list([scols[l] for l in reversed(range(d))])
    f_mat = np.asarray(tcol.T @ vals)
    return np.asarray(C.T @ f_mat.T).T.reshape(-1)


def pcg(A, b, M_solve, tol):
    """linalg.py:450-499 (returns (x, iterations))."""
    n = b.size
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros(n), 0
    x = np.zeros(n)
    r = b.copy()
    z = M_solve(r)
    p = z.copy()
    rz = r @ z
    for it in range(1, 10 * n + 1):
        Ap = A @ p
        alpha = rz / (p @ Ap)
        x += alpha * p
        r -= alpha * Ap
        if np.linalg.norm(r) / bnorm <= tol:
            return x, it
        z = M_solve(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    raise RuntimeError("pcg did not converge")


def solve_w(st, Wt, Mt, Ms, b, d_e, g, tol):
    """solve_w_system (linalg.py:502-547) with the KroneckerMassPreconditioner (linalg.py:176-203)."""
    Kt = (Wt + b * d_e * Mt).toarray()
    nt = Kt.shape[0]
    if np.all(g == 0.0):
        return np.zeros_like(g), []
    facs = [sla.cho_factor(asm.mass_stiff_adv(s)[0].toarray()) for s in st.spatial]
    d = st.d

    def mass_inv(r):
        x = r.reshape(st.spatial_shape)
        for l in range(d):
            axis = d - 1 - l
            moved = np.moveaxis(x, axis, 0)
            sol = sla.cho_solve(facs[l], moved.reshape(moved.shape[0], -1))
            x = np.moveaxis(sol.reshape(moved.shape), 0, axis)
        return x.reshape(-1)

    Y = sla.lu_solve(sla.lu_factor(Kt), g.reshape(nt, -1))
    X = np.empty_like(Y)
    its = []
    for i in range(nt):
        X[i], it = pcg(Ms, Y[i], mass_inv, tol)
        its.append(it)
    return X.reshape(-1), its


def fixed_point_solve(st, T, D, consts, source=None, u0=None, C_m=1.0, b=0.013, d_e=1.0,
                      stabilization="off", relaxation=0.5, tolerance=1e-4, max_iterations=100,
                      lowrank_tol=0.1, indicator_freeze_tol=0.02, linear_tol=1e-8):
    """solver.py:239-386 (box, iterative, every-sweep indicator) with the lifting of the module
    docstring.  ``u0``: None, a callable on (n, d) points or the N_s lifting coefficients.
    Returns dict(u, w, iterations, increments, gmres, pcg, lift)."""
    lift = None if u0 is None else greville_lift(st.spatial, u0)
    if lift is not None and not np.any(lift):
        lift = None
    nt, ns = st.num_time, st.num_space
    Wf, Mf = full_time_factors(st, T)
    Wt, Mt = sp.csr_matrix(Wf[1:, 1:]), sp.csr_matrix(Mf[1:, 1:])
    sig = np.atleast_1d(np.asarray(D, float))
    Ms, Ks = asm.box_spatial(st.spatial, diffusion=None if sig.size == 1 else sig)
    Dk = float(sig[0]) if sig.size == 1 else 1.0
    react = consts["c1"] * consts["a"]
    P = FastDiag.build(st, T, C_m, Dk, react, sigma=None if sig.size == 1 else sig)
    f = load_vector(st, T, source)
    tau = ostab.compute_tau(st.time) if stabilization == "spline_upwind" else None
    u = np.zeros(st.num_dof)
    w = np.zeros(st.num_dof)
    incs, gms, pcgs = [], [], []
    ind = None
    frozen = None
    for k in range(1, max_iterations + 1):
        su = []
        if stabilization == "spline_upwind":
            if frozen is not None:
                su = frozen
            else:
                fresh = compute_theta(st, T, C_m, D, consts, source, u, w, lift)
                freeze = False
                if ind is not None and relaxation < 1.0:
                    drift = float(np.max(np.abs(fresh - ind)))
                    fresh = relaxation * fresh + (1.0 - relaxation) * ind
                    if indicator_freeze_tol > 0.0 and k > 1 and drift * relaxation <= indicator_freeze_tol:
                        freeze = True
                ind = fresh
                lr = ostab.lowrank_factorize(ostab.indicator_for(st, ind), lowrank_tol)
                su = su_full_terms(tau, lr, st, C_m)
                if freeze:
                    frozen = su
        # full-time Kronecker terms: [1:, 1:] is the operator, [1:, 0] the lifted column
        terms = [(C_m, Wf, Ms), (Dk, Mf, Ks)]
        zero = not np.any(u) and not np.any(w) and lift is None
        corr_full = None
        if zero:
            terms.append((react, Mf, Ms))
        else:
            corr_full = reaction_mass_full(st, T, consts, full_coeffs(st, u, lift), full_coeffs(st, w, None))
        terms += su
        op_terms = [(c, sp.csr_matrix(Tm[1:, 1:]), S) for c, Tm, S in terms]
        corr = None if corr_full is None else sp.csr_matrix(corr_full[ns:, ns:])
        op = asm.KronOp(nt, ns, op_terms, corr)
        rhs = f.copy()
        if lift is not None:
            for c, Tm, S in terms:
                col = np.asarray(Tm[1:, 0].toarray()).ravel()
                rhs -= c * np.kron(col, S @ lift)
            if corr_full is not None:
                rhs -= corr_full[ns:, :ns] @ lift
        ut, nit, _ = krylov.gmres(op, rhs, precond=P, tol=linear_tol)
        gms.append(nit)
        g = b * (sp.kron(Mt, Ms) @ u)
        if lift is not None:
            g += b * np.kron(np.asarray(Mf[1:, 0].toarray()).ravel(), Ms @ lift)
        wt, its = solve_w(st, Wt, Mt, Ms, b, d_e, g, linear_tol)
        pcgs.extend(its)
        un = relaxation * ut + (1.0 - relaxation) * u
        wn = relaxation * wt + (1.0 - relaxation) * w
        inc = float(np.max(np.abs(un - u)))
        incs.append(inc)
        u, w = un, wn
        if inc <= tolerance:
            return dict(u=u, w=w, iterations=k, increments=incs, gmres=gms, pcg=pcgs, lift=lift, converged=True)
    return dict(u=u, w=w, iterations=max_iterations, increments=incs, gmres=gms, pcg=pcgs, lift=lift,
                converged=False)
