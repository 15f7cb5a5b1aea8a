"""Mapped (non-affine) spatial geometries.

``GeometryMap`` restates the reference's tensor-product spline map
(geometry.py:31-206): control net in colexicographic order (direction 1
fastest), values and Jacobians on tensor grids of parametric points.
``load_geometry`` / ``save_geometry`` read and write the reference's plain-text
control-point format (geometry.py:309-344), so a geometry built with the
reference (e.g. its ellipse annulus) is used unchanged here.

``MappedSpatialData`` is the host side of the reference's
SpatialQuadratureData (assembly.py:137-219) as the device path needs it:
q = p+1 Gauss rules on the solution mesh, per-direction basis tables, and
at every tensor quadrature point the weight w |det J| and the pulled-back
metric J^-1 J^-T.  The spatial mass / stiffness stencils, the reaction
weight and the load vector are generated from these on the device; the
reference assembles N_s x N_s CSR matrices instead.
"""

import numpy as np


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _einsum(expr, *ops):
    """np.einsum for per-Gauss-point small-tensor contractions over millions of points: numpy's c_einsum
    is single-threaded there (0.2 s a call at 128^3 points), so on a CUDA machine the contraction runs
    through torch on the device and comes back as numpy (setup data; the values agree to rounding)."""
    import torch
    if torch.cuda.is_available() and max(np.asarray(o).size for o in ops) >= (1 << 16):
        dev = torch.device("cuda", torch.cuda.current_device())
        out = torch.einsum(expr, *[torch.as_tensor(np.ascontiguousarray(o), device=dev) for o in ops])
        return out.cpu().numpy()
    return np.einsum(expr, *ops)         # host-only runs (the CPU test suite) and small arrays


from .spaces import SplineSpace, basis_table, gauss_rule

SINGULAR_REL_TOL = 1e-12


class GeometryError(RuntimeError):
    """Singular or invalid geometry map (geometry.py:27-28)."""


class GeometryMap:
    """Tensor-product spline map from [0, 1]^d to the physical domain (geometry.py:31-66)."""

    def __init__(self, spaces, control_points, final_time=1.0, affine_scales=None):
        self.spaces = tuple(spaces)
        self.dim = len(self.spaces)
        n = int(np.prod([s.dimension for s in self.spaces]))
        cp = np.asarray(control_points, dtype=float)
        if cp.shape != (n, self.dim):
            raise ValueError("control_points must have shape (%d, %d)" % (n, self.dim))
        if final_time <= 0:
            raise ValueError("final_time must be positive")
        self.control_points = cp
        self.final_time = float(final_time)
        self.affine_scales = affine_scales
        self._grid = cp.reshape(tuple(s.dimension for s in reversed(self.spaces)) + (self.dim,))

    def grid_data(self, axes, order=1, device=None):
        """x (grid + (d,)) and, for order >= 1, jac (grid + (d, d)) with jac[..., c, a] = dF_c/deta_a,
        for order 2 (host only) hess (grid + (d, d, d)); grid axes in C order (direction d first),
        like geometry.py:135-186.  With a CUDA ``device``
        the tensor contractions run there and torch tensors are returned."""
        if order > 2 or (order == 2 and device is not None):
            raise NotImplementedError("Hessians are evaluated on the host only (residual indicator)")
        d = self.dim
        tabs = [[basis_table(s, np.asarray(ax, float), o) if o <= s.degree else
                 np.zeros((np.asarray(ax).size, s.dimension)) for o in range(order + 1)]
                for s, ax in zip(self.spaces, axes)]
        if device is not None:
            import torch
            tabs = [[torch.from_numpy(np.array(t)).to(device) for t in tl] for tl in tabs]
            grid0 = torch.from_numpy(np.ascontiguousarray(self._grid)).to(device)

            def tabulate(orders):
                val = grid0
                for l in range(d):
                    ax = d - 1 - l
                    val = torch.movedim(torch.tensordot(tabs[l][orders[l]], val, dims=([1], [ax])), 0, ax)
                return val

            out = {"x": tabulate([0] * d)}
            if order >= 1:
                out["jac"] = torch.stack([tabulate([1 if l == a else 0 for l in range(d)]) for a in range(d)], dim=-1)
            return out

        def tabulate(orders):
            val = self._grid
            for l in range(d):
                ax = d - 1 - l
                val = np.moveaxis(np.tensordot(tabs[l][orders[l]], val, axes=(1, ax)), 0, ax)
            return val

        out = {"x": tabulate([0] * d)}
        if order >= 1:
            jac = np.empty(out["x"].shape[:-1] + (d, d))
            for a in range(d):
                orders = [0] * d
                orders[a] = 1
                jac[..., a] = tabulate(orders)
            out["jac"] = jac
        if order >= 2:
            # hess[..., a, b, c] = d^2 F_c / deta_a deta_b (geometry.py:176-184)
            hess = np.empty(out["x"].shape[:-1] + (d, d, d))
            for a in range(d):
                for b in range(a, d):
                    orders = [0] * d
                    orders[a] += 1
                    orders[b] += 1
                    hess[..., a, b, :] = hess[..., b, a, :] = tabulate(orders)
            out["hess"] = hess
        return out


def jacobian_inverse_and_det(jac):
    """Inverse Jacobians and determinants of a grid of maps (the pull-back of geometry.py:207-214).

    A point counts as singular when |det J| falls below SINGULAR_REL_TOL times the product of the
    column norms of J (a scale-free test: a nearly degenerate but large map is still caught)."""
    det = np.linalg.det(jac)
    col_norms = np.linalg.norm(jac, axis=-2)
    bound = SINGULAR_REL_TOL * np.maximum(np.prod(col_norms, axis=-1), 1e-300)
    if (np.abs(det) < bound).any():
        raise GeometryError("singular Jacobian encountered during pull-back")
    return np.linalg.inv(jac), det


def _format_row(values):
    return " ".join(repr(float(v)) for v in values)


def save_geometry(geo, path):
    """Write a GeometryMap in the reference's plain-text layout (geometry.py:309-323), which
    load_geometry (ours and the reference's) reads back bit for bit: a line with d, a line of
    degrees, a line of knot counts, one line of knots per direction, then one control point per line
    (direction 1 fastest)."""
    header = [str(geo.dim),
              " ".join(str(sp.degree) for sp in geo.spaces),
              " ".join(str(len(sp.knots)) for sp in geo.spaces)]
    body = [_format_row(sp.knots) for sp in geo.spaces] + [_format_row(pt) for pt in geo.control_points]
    with open(path, "w") as fh:
        fh.writelines(line + "\n" for line in header + body)


def load_geometry(path, final_time=1.0):
    """Read the plain-text layout of save_geometry (geometry.py:326-344); blank lines and lines
    starting with '#' are skipped."""
    with open(path) as fh:
        rows = [line.split() for line in fh if line.strip() and not line.lstrip().startswith("#")]
    it = iter(rows)
    dim = int(next(it)[0])
    degrees = [int(v) for v in next(it)[:dim]]
    counts = [int(v) for v in next(it)[:dim]]
    spaces = []
    for l in range(dim):
        knots = np.asarray(next(it)[:counts[l]], dtype=float)
        spaces.append(SplineSpace(knots, degrees[l]))
    ncp = int(np.prod([sp.dimension for sp in spaces]))
    ctrl = [row[:dim] for row in it][:ncp]
    if len(ctrl) != ncp:
        raise ValueError("geometry file has %d control rows, expected %d" % (len(ctrl), ncp))
    return GeometryMap(spaces, np.asarray(ctrl, dtype=float), final_time=final_time)


def is_mapped(geometry):
    return isinstance(geometry, GeometryMap) and geometry.affine_scales is None


class FibreConductivity:
    """Transversely isotropic conductivity D(x) = sigma_t I + (sigma_l - sigma_t) f f^T with the fibre
    f(x) the unit physical tangent of map direction ``direction`` (BASELINE cfg 5: fibre-aligned
    sigma_l = 1e-3, sigma_t = 3e-4).  An extension: the reference takes a scalar D (solver.py:66-101,
    assembly.py:205-219); with this object the pulled-back stiffness metric becomes J^-1 D J^-T."""

    def __init__(self, sigma_l, sigma_t, direction=0):
        if sigma_l < 0 or sigma_t < 0:
            raise ValueError("conductivities must be nonnegative")
        self.sigma_l, self.sigma_t, self.direction = float(sigma_l), float(sigma_t), int(direction)

    def tensor(self, jac):
        """D on a grid of Jacobians jac[..., c, a] = dF_c / deta_a: grid + (d, d) (numpy or torch)."""
        f = jac[..., :, self.direction]
        d = jac.shape[-1]
        if isinstance(jac, np.ndarray):
            f = f / np.linalg.norm(f, axis=-1, keepdims=True)
            return self.sigma_t * np.eye(d) + (self.sigma_l - self.sigma_t) * (f[..., :, None] * f[..., None, :])
        import torch
        f = f / torch.linalg.norm(f, dim=-1, keepdim=True)
        eye = torch.eye(d, dtype=jac.dtype, device=jac.device)
        return self.sigma_t * eye + (self.sigma_l - self.sigma_t) * (f[..., :, None] * f[..., None, :])


    def diffusion_coefficients(self, jac, hess, jinv):
        """(MD, divD) for the strong residual's div(D grad u) on a grid of Gauss points (host numpy):
        div(D grad u) = sum_ab MD_ab (d_ab u - sum_e H_abe g_e) + sum_d divD_d g_d with g = J^-T grad_eta u,
        MD = J^-1 D J^-T (the stiffness metric) and divD_d = sum_c d(D_cd)/dx_c
        = (sigma_l - sigma_t) ((div f) f_d + ((f . grad) f)_d), the fibre's physical derivatives from
        the map Hessian: d_a f = (d_a J_k - f (f . d_a J_k)) / |J_k|, df/dx_c = sum_a J^-1[a, c] d_a f.
        (The extension of stabilization.py:273-295 -- whose D is a scalar -- to the cfg-5 fibres.)"""
        # numpy arrays (host restatement, tests) or torch tensors (the device indicator's setup: millions of
        # Gauss points) -- the same formulas through either library
        if _is_torch(jac):
            import torch
            es, eye = torch.einsum, torch.eye(jac.shape[-1], dtype=jac.dtype, device=jac.device)
        else:
            es, eye = _einsum, np.eye(jac.shape[-1])
        k = self.direction
        Jk = jac[..., :, k]
        nrm = (Jk * Jk).sum(-1)[..., None] ** 0.5
        f = Jk / nrm
        D = self.sigma_t * eye + (self.sigma_l - self.sigma_t) * (f[..., :, None] * f[..., None, :])
        MD = es("...ac,...cd,...bd->...ab", jinv, D, jinv)
        dJk = hess[..., :, k, :]                                        # [a, c] = d_a d_k x_c
        da_f = (dJk - f[..., None, :] * es("...ac,...c->...a", dJk, f)[..., :, None]) / nrm[..., None]
        dfdx = es("...ac,...ad->...cd", jinv, da_f)                    # [c, d] = d f_d / d x_c
        divf = es("...cc->...", dfdx)
        fgradf = es("...c,...cd->...d", f, dfdx)
        divD = (self.sigma_l - self.sigma_t) * (divf[..., None] * f + fgradf)
        return MD, divD


def is_fibre(D):
    return isinstance(D, FibreConductivity)


class MappedSpatialData:
    """Quadrature data of a mapped geometry on the solution mesh (assembly.py:137-219).  With a
    ``conductivity`` (FibreConductivity) the stiffness metric is J^-1 D J^-T instead of J^-1 J^-T."""

    def __init__(self, spatial_spaces, geometry, device="auto", conductivity=None, coefficient_rank=None,
                 coefficient_tol=1e-6):
        """``device``: where the map is evaluated and the Jacobians inverted ("auto": the current
        CUDA device if there is one; None: host numpy).  Results are host arrays either way.
        ``coefficient_rank``: if given, M_s and K_s (and the reaction's |det J|) use canonical rank
        <= coefficient_rank approximations of the coefficients (LowRankCoefficients, BASELINE cfg 5)
        instead of the exact pulled-back values; ``coefficient_tol`` is the relative error at which
        the rank search stops."""
        self.spaces = tuple(spatial_spaces)
        d = len(self.spaces)
        if geometry.dim != d:
            raise ValueError("geometry dimension %d != number of spatial directions %d" % (geometry.dim, d))
        self.geo = geometry
        self.q = [s.degree + 1 for s in self.spaces]
        self.rules = [gauss_rule(s.breakpoints, s.degree + 1) for s in self.spaces]   # (points, weights)
        if device == "auto":
            import torch
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
        if device is not None:
            import torch
            data = geometry.grid_data([r[0] for r in self.rules], order=1, device=device)
            jac = data["jac"]
            det = torch.linalg.det(jac)
            scale = torch.prod(torch.linalg.norm(jac, dim=-2), dim=-1)
            if bool(torch.any(det.abs() < SINGULAR_REL_TOL * torch.clamp(scale, min=1e-300)).item()):
                raise GeometryError("singular Jacobian encountered during pull-back")
            self.xgrid = data["x"].cpu().numpy()
            jinv = torch.linalg.inv(jac)
            self._G = None
            if conductivity is not None:
                self._G = (jinv @ conductivity.tensor(jac) @ jinv.transpose(-1, -2)).cpu().numpy()
            self.jinv = jinv.cpu().numpy()
            self.detj = det.cpu().numpy()
            del data, jac, det, scale, jinv
        else:
            data = geometry.grid_data([r[0] for r in self.rules], order=1)
            self.xgrid = data["x"]
            self.jinv, self.detj = jacobian_inverse_and_det(data["jac"])
            self._G = None
            if conductivity is not None:
                self._G = self.jinv @ conductivity.tensor(data["jac"]) @ np.swapaxes(self.jinv, -1, -2)
        w = np.ones(())
        for l in reversed(range(d)):
            w = np.multiply.outer(w, self.rules[l][1])
        self.wgrid = w                                        # (Q_d, ..., Q_1)
        self.grid_shape = self.wgrid.shape
        self.conductivity = conductivity
        self.lowrank = None
        if coefficient_rank is not None:
            self.lowrank = LowRankCoefficients(self, coefficient_rank, coefficient_tol, device=device)

    def measure(self):
        """w |det J| on the grid."""
        return self.wgrid * np.abs(self.detj)

    def metric(self, a, b):
        """(J^-1 J^-T)_{ab} on the grid ((J^-1 D J^-T)_{ab} with a conductivity)."""
        if self._G is not None:
            return self._G[..., a, b]
        return np.einsum("...k,...k->...", self.jinv[..., a, :], self.jinv[..., b, :])

    def metric_diag(self, direction):
        return self.metric(direction, direction)

    def physical_points(self):
        return self.xgrid.reshape(-1, len(self.spaces))

    def tables(self, l, order):
        """(Q_l, n_l) basis table of direction l (collocation_matrix, assembly.py:157-160)."""
        return basis_table(self.spaces[l], self.rules[l][0], order)


def quad_tables(sd, orders, p, nmax):
    """Basis-product tables of the quadrature channel generator (mi_op_set_quad_channel):
    T[t, l, i, a, b] = B^(o)_i(x_k) B^(o')_j(x_k), j = i + a - p, k = (i - p) q_l + b, for the
    derivative orders ``orders[t][l] = (o, o')`` of term t."""
    d = len(sd.spaces)
    kw = max((p + 1) * q for q in sd.q)
    T = np.zeros((len(orders), d, nmax, 2 * p + 1, kw))
    for l in range(d):
        n, q = sd.spaces[l].dimension, sd.q[l]
        Q = sd.rules[l][0].size
        i = np.arange(n)[:, None, None]
        a = np.arange(2 * p + 1)[None, :, None]
        b = np.arange((p + 1) * q)[None, None, :]
        j = i + a - p
        k = (i - p) * q + b
        ok = (j >= 0) & (j < n) & (k >= 0) & (k < Q)
        jj, kk = np.where(ok, j, 0), np.where(ok, k, 0)
        ii = np.broadcast_to(i, ok.shape)
        tabs = {}
        for t, ords in enumerate(orders):
            oi, oj = ords[l]
            for o in (oi, oj):
                if o not in tabs:
                    tabs[o] = sd.tables(l, o)
            T[t, l, :n, :, :(p + 1) * q] = np.where(ok, tabs[oi][kk, ii] * tabs[oj][kk, jj], 0.0)
    return np.ascontiguousarray(T)


def mass_terms(sd):
    """(coef, theta, orders) of M_s = C^T diag(w |det J|) C (assembly.py:197-203)."""
    d = len(sd.spaces)
    return [(1.0, sd.measure(), [(0, 0)] * d)]


def stiffness_terms(sd, coef=1.0):
    """K_s = sum_ab C_a^T diag(w |det J| (J^-1 J^-T)_ab) C_b (assembly.py:205-219): the test function
    carries the derivative in direction a, the trial function the one in direction b."""
    d = len(sd.spaces)
    base = sd.measure()
    terms = []
    for a in range(d):
        for b in range(d):
            orders = [(1 if l == a else 0, 1 if l == b else 0) for l in range(d)]
            terms.append((coef, base * sd.metric(a, b), orders))
    return terms


def separable_weights(sd):
    """Rank-one per-direction surrogates of the pulled-back measures (FastDiagPreconditioner.
    _separable_weights, linalg.py:228-262): mass[l] approximates |det J| multiplicatively, stiff[l]
    the metric coefficient (J^-1 J^-T)_ll |det J| relative to the other directions' mass weights."""
    d = len(sd.spaces)
    detj = np.abs(sd.detj)
    log_detj = np.log(detj)
    grand = log_detj.mean()
    mass = []
    for l in range(d):
        axis = d - 1 - l
        other = tuple(x for x in range(d) if x != axis)
        main = log_detj.mean(axis=other) if other else log_detj
        mass.append(np.exp(main - grand + grand / d))
    stiff = []
    for l in range(d):
        axis = d - 1 - l
        coeff = detj * sd.metric_diag(l)
        denom = np.ones_like(coeff)
        for m in range(d):
            if m == l:
                continue
            shape = [1] * d
            shape[d - 1 - m] = mass[m].size
            denom = denom * mass[m].reshape(shape)
        ratio = coeff / denom
        other = tuple(x for x in range(d) if x != axis)
        stiff.append(ratio.mean(axis=other) if other else ratio)
    return mass, stiff


def _khatri_rao(A, B):
    """Column-wise Kronecker product: (I, r), (J, r) -> (I*J, r), row i*J + j."""
    return (A[:, None, :] * B[None, :, :]).reshape(-1, A.shape[1])


def _leading_vectors(G, r, gen):
    """r leading eigenvectors of the symmetric Gram matrix G (the HOSVD start of CP-ALS); columns past
    G's size are seeded random."""
    import torch
    _, V = torch.linalg.eigh(G)
    k = min(r, G.shape[0])
    A = V[:, -k:].flip(-1)
    if k < r:
        extra = torch.rand((G.shape[0], r - k), generator=gen, dtype=G.dtype).to(G.device)
        A = torch.cat([A, extra], dim=1)
    return A.contiguous()


def cp_als(X, rank, max_iter=500, rtol=1e-13):
    """Canonical polyadic approximation X ~ sum_r prod_k A_k[:, r] of a 1-, 2- or 3-way torch f64
    array (axis k of X <-> factor k).  1-way: X itself (rank 1); 2-way: truncated SVD (optimal);
    3-way: alternating least squares from the HOSVD start, column norms balanced each sweep, stopped
    when the squared residual changes by less than ``rtol`` relative.  Returns (factors, rel_err) with
    rel_err = ||X - X_r|| / ||X|| evaluated explicitly.  (The low-rank coefficient approximation of
    BASELINE cfg 5 has no counterpart in the reference.)"""
    import torch
    nd = X.dim()
    if float(torch.linalg.norm(X)) == 0.0:
        return [torch.zeros((n, 1), dtype=X.dtype, device=X.device) for n in X.shape], 0.0
    if nd == 1:
        return [X[:, None].clone()], 0.0
    if nd == 2:
        U, S, Vh = torch.linalg.svd(X, full_matrices=False)
        r = min(rank, S.numel())
        A = [U[:, :r] * S[:r], Vh[:r].T.contiguous()]
    elif nd == 3:
        Q0, Q1, Q2 = X.shape
        gen = torch.Generator().manual_seed(0)
        X0 = X.reshape(Q0, Q1 * Q2)
        X2 = X.reshape(Q0 * Q1, Q2)
        A = [_leading_vectors(X0 @ X0.T, rank, gen),
             _leading_vectors(torch.einsum("ijk,ilk->jl", X, X), rank, gen),
             _leading_vectors(X2.T @ X2, rank, gen)]
        nx2 = float((X * X).sum())
        prev = None
        for _ in range(max_iter):
            G = [a.T @ a for a in A]
            A[0] = (X0 @ _khatri_rao(A[1], A[2])) @ torch.linalg.pinv(G[1] * G[2], hermitian=True)
            G[0] = A[0].T @ A[0]
            T = (X2 @ A[2]).reshape(Q0, Q1, -1)
            A[1] = torch.einsum("ijr,ir->jr", T, A[0]) @ torch.linalg.pinv(G[0] * G[2], hermitian=True)
            G[1] = A[1].T @ A[1]
            V = G[0] * G[1]
            M = X2.T @ _khatri_rao(A[0], A[1])
            A[2] = M @ torch.linalg.pinv(V, hermitian=True)
            res2 = max(nx2 - 2.0 * float((M * A[2]).sum()) + float((V * (A[2].T @ A[2])).sum()), 0.0)
            nrm = [torch.linalg.norm(a, dim=0) for a in A]
            g = (nrm[0] * nrm[1] * nrm[2]).clamp_min(1e-300) ** (1.0 / 3.0)
            A = [a * (g / n.clamp_min(1e-300)) for a, n in zip(A, nrm)]
            if prev is not None and abs(prev - res2) <= rtol * max(prev, 1e-30 * nx2):
                break
            prev = res2
    else:
        raise ValueError("cp_als takes 1-, 2- or 3-way arrays")
    err = float(torch.linalg.norm(X - cp_reconstruct(A)) / torch.linalg.norm(X).clamp_min(1e-300))
    return A, err


def cp_reconstruct(A):
    """sum_r prod_k A_k[:, r] as a dense array (axis k <-> A[k])."""
    import torch
    if len(A) == 1:
        return A[0].sum(dim=1)
    if len(A) == 2:
        return A[0] @ A[1].T
    return torch.einsum("ir,jr,kr->ijk", A[0], A[1], A[2])


class LowRankCoefficients:
    """Canonical rank <= ``max_rank`` approximations of the pulled-back geometry and conductivity
    coefficients on the Gauss grid (BASELINE cfg 5: "geometry and conductivity coefficients low-rank
    approximated (canonical rank <= 8)"; absent in the reference, whose SpatialQuadratureData integrates
    the exact coefficients, assembly.py:197-219):

    * ``"mass"``: |det J|,
    * ``(a, b)``, a <= b: |det J| (J^-1 D J^-T)_ab (D = I, or the FibreConductivity tensor).

    Each field c is approximated by c ~ sum_r prod_l g_{l,r}(xi_l) with the smallest rank whose
    relative error on the grid is <= ``tol`` (capped at ``max_rank``).  Then every quadrature term of
    M_s / K_s is a sum of Kronecker products of 1D weighted matrices
    F_{l,r}[i, j] = sum_k w_k g_{l,r}(xi_k) B^(o)_i(xi_k) B^(o')_j(xi_k), so the device builds the
    stencils with the Kronecker generator (mi_op_set_kron_channel) instead of tensor quadrature."""

    def __init__(self, sd, max_rank=8, tol=1e-6, device="auto"):
        import torch
        if max_rank < 1:
            raise ValueError("max_rank must be >= 1")
        if device == "auto":
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
        dev = torch.device("cpu") if device is None else torch.device(device)
        d = len(sd.spaces)
        self.d, self.max_rank, self.tol = d, int(max_rank), float(tol)
        detj = np.abs(sd.detj)
        fields = {"mass": detj}
        for a in range(d):
            for b in range(a, d):
                fields[(a, b)] = detj * sd.metric(a, b)
        self.factors, self.rank, self.error = {}, {}, {}
        for key, f in fields.items():
            X = torch.as_tensor(np.ascontiguousarray(f), dtype=torch.float64, device=dev)
            for r in range(1, self.max_rank + 1):
                A, err = cp_als(X, r)
                if err <= self.tol:
                    break
            # factor of direction l = array axis d-1-l
            self.factors[key] = [A[d - 1 - l].cpu().numpy() for l in range(d)]
            self.rank[key] = A[0].shape[1]
            self.error[key] = err
            del X

    def reconstruct(self, key):
        """The rank-r field on the grid (Q_d, ..., Q_1)."""
        import torch
        A = [torch.as_tensor(self.factors[key][self.d - 1 - k]) for k in range(self.d)]
        return cp_reconstruct(A).numpy()

    def stiffness_key(self, a, b):
        return (min(a, b), max(a, b))

    def kron_terms(self, sd, kind, p, nmax):
        """(coef, bands) of mi_op_set_kron_channel for ``kind`` "mass" (M_s) or "stiffness" (K_s, the
        test function carrying the derivative in direction a, the trial function in b, as
        stiffness_terms)."""
        from .spaces import to_band
        d = self.d
        if kind == "mass":
            terms = [("mass", [(0, 0)] * d)]
        elif kind == "stiffness":
            terms = [(self.stiffness_key(a, b), [(1 if l == a else 0, 1 if l == b else 0) for l in range(d)])
                     for a in range(d) for b in range(d)]
        else:
            raise ValueError("kind must be 'mass' or 'stiffness'")
        rows = []
        for key, orders in terms:
            g = self.factors[key]
            for r in range(g[0].shape[1]):
                row = []
                for l in range(d):
                    oi, oj = orders[l]
                    w = sd.rules[l][1] * g[l][:, r]
                    F = (sd.tables(l, oi) * w[:, None]).T @ sd.tables(l, oj)
                    row.append(to_band(F, p))
                rows.append(row)
        bands = np.zeros((len(rows), d, nmax, 2 * p + 1))
        for t, row in enumerate(rows):
            for l in range(d):
                bands[t, l, :row[l].shape[0]] = row[l]
        return np.ones(len(rows)), np.ascontiguousarray(bands)

    def summary(self):
        return {("%s" % (k,)).replace(" ", ""): {"rank": self.rank[k], "rel_err": self.error[k]}
                for k in self.factors}


def interpolate_map(spaces, fn):
    """Tensor-product spline map interpolating fn: (m, d) parametric -> (m, d) physical at the Greville
    points (collocation solve per direction)."""
    from .spaces import greville
    d = len(spaces)
    g = [greville(s) for s in spaces]
    mesh = np.meshgrid(*[g[l] for l in reversed(range(d))], indexing="ij")
    pts = np.stack([mesh[d - 1 - l].ravel() for l in range(d)], axis=-1)
    X = np.asarray(fn(pts), float).reshape(tuple(s.dimension for s in reversed(spaces)) + (d,))
    for l in range(d):
        C = basis_table(spaces[l], g[l], 0)
        ax = d - 1 - l
        X = np.moveaxis(np.tensordot(np.linalg.inv(C), X, axes=(1, ax)), 0, ax)
    return GeometryMap(spaces, X.reshape(-1, d))


def prolate_shell_geometry(final_time=1.0, radii=(1.0, 1.0, 2.0), thickness=0.2, polar=(np.pi / 6, 5 * np.pi / 6),
                           degree=3, elements=8):
    """BASELINE cfg 5 geometry (absent from the reference): a thick slab of a
    prolate-ellipsoid shell, quarter sector in azimuth, as a degree-3 tensor-product spline map
    interpolating the exact shell at the Greville points.  Direction 1: azimuth phi in [0, pi/2],
    direction 2: polar angle theta in ``polar``, direction 3: through the wall, rho in
    [1 - thickness, 1] (x = rho (a sin(theta) cos(phi), b sin(theta) sin(phi), c cos(theta)))."""
    a, b, c = radii
    t0, t1 = polar

    def shell(p):
        phi = 0.5 * np.pi * p[:, 0]
        th = t1 - (t1 - t0) * p[:, 1]                 # decreasing theta keeps det J > 0
        rho = 1.0 - thickness + thickness * p[:, 2]
        return np.stack([rho * a * np.sin(th) * np.cos(phi), rho * b * np.sin(th) * np.sin(phi),
                         rho * c * np.cos(th)], axis=1)

    spaces = [SplineSpace.uniform(degree, elements) for _ in range(3)]
    geo = interpolate_map(spaces, shell)
    geo.final_time = float(final_time)
    return geo


class MappedSUData:
    """Quadrature data of the Spline Upwind spatial factors S^s_r on a mapped geometry
    (assemble_stabilization, stabilization.py:469-488: SpatialQuadratureData with p+2 Gauss points on
    cells split at the spatial Greville abscissae, assembly.py:137-203, weight w |det J| times the
    multilinear profile theta_r of LowRankIndicator.space_profile, stabilization.py:383-398).

    The refined rule has a variable number of Gauss points per element, so every basis function i
    of direction l gets an explicit window kst[l][i] .. kst[l][i] + kw[l] - 1 of that direction's
    points (mi_op_set_quad_channel_k)."""

    def __init__(self, spatial_spaces, geometry, device="auto"):
        from .factors import hat_values
        from .spaces import cells_with, greville
        self.spaces = tuple(spatial_spaces)
        d = len(self.spaces)
        self.grev = [greville(s) for s in self.spaces]
        self.rules = [gauss_rule(cells_with(s, g), s.degree + 2) for s, g in zip(self.spaces, self.grev)]
        axes = [r[0] for r in self.rules]
        if device == "auto":
            import torch
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
        if device is not None:
            import torch
            jac = geometry.grid_data(axes, order=1, device=device)["jac"]
            det = torch.linalg.det(jac).abs().cpu().numpy()
            del jac
        else:
            det = np.abs(np.linalg.det(geometry.grid_data(axes, order=1)["jac"]))
        w = np.ones(())
        for l in reversed(range(d)):
            w = np.multiply.outer(w, self.rules[l][1])
        self.measure = w * det                              # (Q_d, ..., Q_1)
        self.Q = [r[0].size for r in self.rules]
        self.kst, self.kend = [], []
        for s, (x, _) in zip(self.spaces, self.rules):
            p, u = s.degree, np.asarray(s.knots, float)
            i = np.arange(s.dimension)
            self.kst.append(np.searchsorted(x, u[i]).astype(np.int32))
            self.kend.append(np.searchsorted(x, u[i + p + 1]).astype(np.int32))
        self.kw = [int(np.max(b - a)) for a, b in zip(self.kst, self.kend)]
        self.hats = [hat_values(g, x) for g, (x, _) in zip(self.grev, self.rules)]

    def tables(self, p, nmax):
        """T[0, l, i, a, b] = B_i(x_k) B_j(x_k), j = i + a - p, k = kst[l][i] + b (one mass term)."""
        d = len(self.spaces)
        kw = max(self.kw)
        T = np.zeros((1, d, nmax, 2 * p + 1, kw))
        for l, s in enumerate(self.spaces):
            n, x = s.dimension, self.rules[l][0]
            B = basis_table(s, x, 0)
            i = np.arange(n)[:, None, None]
            a = np.arange(2 * p + 1)[None, :, None]
            b = np.arange(kw)[None, None, :]
            j = i + a - p
            k = self.kst[l][:, None, None] + b
            ok = (j >= 0) & (j < n) & (k < self.kend[l][:, None, None])
            jj, kk = np.where(ok, j, 0), np.where(ok, k, 0)
            T[0, l, :n] = np.where(ok, B[kk, np.broadcast_to(i, ok.shape)] * B[kk, jj], 0.0)
        return np.ascontiguousarray(T)

    def kstart(self, nmax):
        ks = np.zeros((len(self.spaces), nmax), dtype=np.int32)
        for l, k in enumerate(self.kst):
            ks[l, :k.size] = k
        return ks

    def weight(self, theta_r):
        """w |det J| times the multilinear interpolant of theta_r (flat N_s, direction 1 fastest) on
        the Greville grid, at the refined Gauss grid (C order, direction d first)."""
        d = len(self.spaces)
        prof = np.asarray(theta_r, float).reshape(tuple(s.dimension for s in reversed(self.spaces)))
        for l in range(d):
            ax = d - 1 - l
            prof = np.moveaxis(np.tensordot(self.hats[l], prof, axes=(1, ax)), 0, ax)
        return self.measure * prof
