"""Problem description and per-sweep host setup of the fixed-point driver.

Mirrors the reference's ``MonodomainProblem`` / ``FixedPointConfig`` /
``SolveResult`` / ``FixedPointDiverged`` (solver.py:58-160) and the two
per-sweep host computations the driver needs on box geometries:

* ``load_vector``: the source load vector of rhs_vectors (assembly.py:350-398);
* ``compute_theta``: the Spline Upwind residual indicator
  (stabilization.py:235-339) -- strong residual with the Rogers-McCulloch
  ionic current at the Gauss points, element maxima, support-extension
  window maxima, clamped ratio.

Both are host numpy (sum factorised); the (d+1)-way solve they feed runs on
the device.  Geometry: axis-aligned boxes (the reference's affine maps).
"""

import os
import warnings
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from .spaces import basis_table, gauss_rule, greville


SOURCE_THREADS = max(1, min(32, os.cpu_count() or 1))   # host threads for source evaluation


class DeviceSource:
    """A source term f(x, t) with a device implementation.

    Called like the reference's source callable (numpy points (Q, d) and times (Q,) -> (Q,)), so
    the reference and the oracle see the same function.  ``torch`` is the same function on torch
    tensors; when present, the Gauss-point values that feed the load vector and the residual
    indicator are evaluated and contracted on the GPU instead of on the host."""

    def __init__(self, host, torch):
        self.host = host
        self.torch = torch

    def __call__(self, x, t):
        return self.host(x, t)


def device_capable(source):
    return source is not None and callable(getattr(source, "torch", None))


class FixedPointDiverged(RuntimeError):
    """Fixed-point iteration exhausted its budget; carries the last state."""

    def __init__(self, message, result):
        super().__init__(message)
        self.result = result


class BoxGeometry:
    """Axis-aligned box prod_l (o_l, o_l + L_l) x (0, T) (geometry.py:217-234)."""

    def __init__(self, lengths, final_time=1.0, offsets=None):
        self.lengths = np.atleast_1d(np.asarray(lengths, float))
        self.dim = self.lengths.size
        self.offsets = np.zeros(self.dim) if offsets is None else np.atleast_1d(np.asarray(offsets, float))
        if final_time <= 0:
            raise ValueError("final_time must be positive")
        self.final_time = float(final_time)
        self.affine_scales = (self.lengths, self.offsets)


def box_of(geometry):
    """(lengths, offsets) of a box geometry (ours or the reference's GeometryMap)."""
    aff = getattr(geometry, "affine_scales", None)
    if aff is None:
        raise NotImplementedError("mapped (non-affine) geometries are not supported on the device path")
    L, off = aff
    return np.asarray(L, float), np.asarray(off, float)


@dataclass
class MonodomainProblem:
    """solver.py:66-101 (same fields, defaults and validation)."""

    geometry: object
    space: object
    source: object = None
    C_m: float = 1.0
    D: float = 1e-4
    a: float = 0.13
    b: float = 0.013
    c1: float = 0.26
    c2: float = 0.1
    d_e: float = 1.0
    # extension (BASELINE's stimuli; absent in the reference): initial potential u0 as a
    # callable on (n, d) physical points or as N_s spline coefficients; lifted as u0_h(x) b_0(t) with
    # u0_h the Greville quasi-interpolant (lift_coefficients).  None = the reference (u vanishes at t=0).
    u0: object = None

    def __post_init__(self):
        for name in ("C_m", "a", "b", "c1", "c2", "d_e"):
            if getattr(self, name) < 0:
                raise ValueError("%s must be nonnegative" % name)
        # D: scalar (the reference) or one value per spatial direction (anisotropic diagonal sigma,
        # the oracle extension of SURVEY Appendix B)
        # or a geometry.FibreConductivity on mapped geometries (BASELINE cfg 5 extension)
        from .geometry import is_fibre, is_mapped
        if is_fibre(self.D):
            if not is_mapped(self.geometry):
                raise ValueError("a fibre conductivity needs a mapped geometry")
        else:
            Dv = np.atleast_1d(np.asarray(self.D, float))
            if np.any(Dv < 0):
                raise ValueError("D must be nonnegative")
            if Dv.size not in (1, len(self.space.spatial)):
                raise ValueError("D must be a scalar or one value per spatial direction")
        if self.geometry.final_time <= 0:
            raise ValueError("final time must be positive")
        if self.geometry.dim != len(self.space.spatial):
            raise ValueError("geometry and space dimensions differ")

    @property
    def final_time(self):
        return self.geometry.final_time

    def scalar_D(self):
        """The scalar multiplying K_s: D itself, or 1 when a FibreConductivity is folded into K_s."""
        from .geometry import is_fibre
        return 1.0 if is_fibre(self.D) else self.D

    def diffusion(self):
        """Per-direction diffusion coefficients (length d)."""
        Dv = np.atleast_1d(np.asarray(self.D, float))
        return np.repeat(Dv, len(self.space.spatial)) if Dv.size == 1 else Dv

    def reaction_constants(self):
        return {"c1": self.c1, "a": self.a, "c2": self.c2}


def lift_coefficients(problem):
    """N_s coefficients of u0_h = sum_s u0(F(gamma_s)) B_s (Schoenberg quasi-interpolant at the tensor
    Greville abscissae gamma_s, mapped to physical points): monotone, so a step u0 stays in its range.
    None when the problem has no (or a zero) u0."""
    from .spaces import greville_points
    u0 = problem.u0
    if u0 is None:
        return None
    st = problem.space
    if callable(u0):
        eta = greville_points(st.spatial)
        aff = getattr(problem.geometry, "affine_scales", None)
        if aff is not None:
            L, off = aff
            x = np.asarray(off, float)[None, :] + eta * np.asarray(L, float)[None, :]
        else:
            d = len(st.spatial)
            axes = [greville(s) for s in st.spatial]
            x = np.asarray(problem.geometry.grid_data(axes, order=0)["x"]).reshape(-1, d)
        c = np.asarray(u0(x), float).reshape(-1)
    else:
        c = np.asarray(u0, float).reshape(-1)
    if c.size != st.num_space:
        raise ValueError("u0 needs one coefficient per spatial function (%d), got %d" % (st.num_space, c.size))
    return None if not np.any(c) else c


@dataclass
class FixedPointConfig:
    """solver.py:104-137.  ``linear_solver`` "auto" selects the device GMRES
    (the reference's direct LU for N <= 20000 is host-only and out of scope);
    "direct" is rejected."""

    relaxation: float = 0.5
    tolerance: float = 1e-4
    max_iterations: int = 100
    stabilization: str = "off"
    lowrank_tol: float = 0.1
    indicator_update: str = "every_sweep"
    indicator_freeze_tol: float = 0.02
    linear_solver: str = "auto"
    linear_tol: float = 1e-8
    evolve_recovery: bool = True
    indicator_override: object = None
    verbose: bool = False
    # extension (BASELINE cfg 5; not in the reference): canonical rank <= coefficient_rank approximations
    # of the mapped geometry / conductivity coefficients in M_s, K_s (geometry.LowRankCoefficients);
    # None keeps the exact pulled-back coefficients of the reference
    coefficient_rank: object = None
    coefficient_tol: float = 1e-6

    def __post_init__(self):
        if not 0.0 < self.relaxation <= 1.0:
            raise ValueError("relaxation must lie in (0, 1]")
        if self.tolerance <= 0:
            raise ValueError("tolerance must be positive")
        if self.stabilization not in ("off", "spline_upwind"):
            raise ValueError("unknown stabilization %r" % self.stabilization)
        if self.indicator_update not in ("every_sweep", "frozen"):
            raise ValueError("unknown indicator update %r" % self.indicator_update)
        if self.linear_solver not in ("auto", "direct", "iterative"):
            raise ValueError("unknown linear solver %r" % self.linear_solver)
        if self.coefficient_rank is not None and int(self.coefficient_rank) < 1:
            raise ValueError("coefficient_rank must be >= 1")


@dataclass
class SolveResult:
    """solver.py:140-160."""

    u: np.ndarray
    w: np.ndarray
    iterations: int
    increments: list = field(default_factory=list)
    converged: bool = True
    gmres_iterations: list = field(default_factory=list)
    pcg_iterations: list = field(default_factory=list)
    wall_time: float = 0.0
    indicator: object = None
    phase_seconds: dict = field(default_factory=dict)   # device driver only: wall time per phase
    lift: object = None   # u0 lifting coefficients (N_s) when the problem has u0: u_h = lift b_0 + u

    @property
    def avg_gmres(self):
        return float(np.mean(self.gmres_iterations)) if self.gmres_iterations else 0.0

    @property
    def avg_pcg(self):
        return float(np.mean(self.pcg_iterations)) if self.pcg_iterations else 0.0


class ResidualIndicator:
    """N_t x N_s indicator values with the Greville grids (stabilization.py:177-193)."""

    def __init__(self, values, time_greville, spatial_grevilles, spatial_shape):
        # numpy, or a CUDA tensor when the driver keeps the indicator on the device
        self.values = values if _is_tensor(values) else np.asarray(values, float)
        self.time_greville = np.asarray(time_greville, float)
        self.spatial_grevilles = [np.asarray(g, float) for g in spatial_grevilles]
        self.spatial_shape = tuple(spatial_shape)

    @property
    def max(self):
        if _is_tensor(self.values):
            return float(self.values.max().item()) if self.values.numel() else 0.0
        return float(self.values.max(initial=0.0))


def _is_tensor(v):
    return type(v).__module__.startswith("torch")


# --------------------------------------------------------------------------
# Gauss-grid helpers (default q = p+1 rules on the breakpoints)
# --------------------------------------------------------------------------

def _mode(A, X, axis):
    if not isinstance(X, np.ndarray):                 # torch tensor (device load vector)
        import torch
        At = torch.tensor(A, dtype=X.dtype, device=X.device)    # copies (A may be a read-only table)
        return torch.movedim(torch.tensordot(At, X, dims=([1], [axis])), 0, axis)
    t = np.moveaxis(X, axis, 0)
    out = (A @ t.reshape(t.shape[0], -1)).reshape((A.shape[0],) + t.shape[1:])
    return np.moveaxis(out, 0, axis)


class GaussGrid:
    """Default Gauss rules (q = p+1) of every direction with basis tables."""

    def __init__(self, st, geometry, mapped=None):
        from .geometry import MappedSpatialData, is_mapped
        self.st = st
        # mapped geometries: parametric rules, physical points and |det J| from the map
        if mapped is None and is_mapped(geometry):
            mapped = MappedSpatialData(st.spatial, geometry)
        self.mapped = mapped
        if self.mapped is None:
            self.L, self.off = box_of(geometry)
        else:
            self.L, self.off = np.ones(len(st.spatial)), np.zeros(len(st.spatial))
        self.T = geometry.final_time
        self.d = len(st.spatial)
        self.sx, self.sw, self.sB = [], [], []
        for s in st.spatial:
            x, w = gauss_rule(s.breakpoints, s.degree + 1)
            self.sx.append(x)
            self.sw.append(w)
            self.sB.append([basis_table(s, x, o) for o in range(min(2, s.degree) + 1)])
        tx, tw = gauss_rule(st.time.breakpoints, st.time.degree + 1)
        self.tx, self.tw = tx, tw
        self.tB = [basis_table(st.time, tx, o)[:, 1:] for o in range(2)]   # constrained time basis
        self.tB0 = [basis_table(st.time, tx, o)[:, 0].copy() for o in range(2)]   # the dropped b_0 (lifting)

    def field(self, coeffs, space_orders, time_order):
        """Values on the grid (Q_t, Q_d, ..., Q_1) of a coefficient vector."""
        st, d = self.st, self.d
        U = np.asarray(coeffs, float).reshape(st.coeff_shape)
        out = _mode(self.tB[time_order], U, 0)
        for l in range(d):
            out = _mode(self.sB[l][space_orders[l]], out, 1 + (d - 1 - l))
        return out

    def physical_points(self):
        if self.mapped is not None:
            return self.mapped.physical_points()
        d = self.d
        mesh = np.meshgrid(*[self.off[l] + self.L[l] * self.sx[l] for l in reversed(range(d))], indexing="ij")
        return np.stack([mesh[d - 1 - l].ravel() for l in range(d)], axis=-1)

    def source_values(self, source):
        return self.source_rows(source, 0, self.tx.size)

    def source_chunks(self, source, rows_per_chunk):
        """Yield (i0, i1, values) over all time Gauss rows, rows_per_chunk at a time."""
        nq = self.tx.size
        for i0 in range(0, nq, rows_per_chunk):
            i1 = min(nq, i0 + rows_per_chunk)
            yield i0, i1, self.source_rows(source, i0, i1)

    def source_rows_device(self, source, i0, i1, device):
        """Like source_rows, evaluated on the device by ``source.torch`` (one call per time point)."""
        import torch
        if getattr(self, "_xq_dev", None) is None or self._xq_dev.device != torch.device(device):
            self._xq_dev = torch.from_numpy(self.physical_points()).to(device)
        xq = self._xq_dev
        qs = xq.shape[0]
        tq = self.tx[i0:i1] * self.T
        fv = torch.empty((tq.size, qs), dtype=torch.float64, device=xq.device)
        for i in range(tq.size):
            fv[i] = torch.as_tensor(source.torch(xq, torch.full((qs,), float(tq[i]), dtype=torch.float64,
                                                                device=xq.device)),
                                    dtype=torch.float64).reshape(qs)
        return fv.reshape((tq.size,) + tuple(x.size for x in reversed(self.sx)))

    def source_rows(self, source, i0, i1):
        """Source at time Gauss points i0..i1-1 x all spatial Gauss points, (i1-i0, Q_d, ..., Q_1)."""
        if getattr(self, "_xq", None) is None:
            self._xq = self.physical_points()
        xq = self._xq
        qs = xq.shape[0]
        tq = self.tx[i0:i1] * self.T
        fv = np.empty((tq.size, qs))

        def row(i):
            fv[i] = np.asarray(source(xq, np.full(qs, tq[i])), float).reshape(qs)

        # one call per time point like the reference (assembly.py:380-388); numpy releases the GIL,
        # so large grids evaluate on a thread pool (the source must be a pure function of (x, t))
        workers = min(SOURCE_THREADS, tq.size) if qs * tq.size >= (1 << 22) else 1
        if workers > 1:
            with ThreadPoolExecutor(max_workers=workers) as pool:
                list(pool.map(row, range(tq.size)))
        else:
            for i in range(tq.size):
                row(i)
        return fv.reshape((tq.size,) + tuple(x.size for x in reversed(self.sx)))


def load_vector(st, geometry, source, grid=None, chunk_points=1 << 24, chunks=None, device=None):
    """f_vec[i] = int int f B_i (assembly.py:350-398, box geometry).  The Gauss grid is visited in
    chunks of time points (spatial projection per chunk, then the time projection accumulates),
    so the full space-time grid is never held at once; time points where the source vanishes
    identically contribute nothing and are skipped.  ``chunks`` may supply the evaluated source
    as (i0, i1, values) rows (GaussGrid.source_chunks) so another consumer can share them.
    A DeviceSource is evaluated and contracted on the GPU; the result is then a device tensor."""
    if source is None:
        return np.zeros(st.num_dof)
    g = grid if grid is not None else GaussGrid(st, geometry)
    d = g.d
    if g.mapped is not None:
        ws = g.mapped.measure()                        # w |det J| (rhs_vectors, assembly.py:385-387)
    else:
        ws = np.asarray(g.sw[d - 1] * g.L[d - 1])
        for l in reversed(range(d - 1)):
            ws = np.multiply.outer(ws, g.sw[l] * g.L[l])
    if chunks is None:
        rows_per = max(1, chunk_points // max(1, ws.size))
        if device_capable(source):
            import torch
            dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
            nq = g.tx.size
            chunks = ((i0, min(nq, i0 + rows_per), g.source_rows_device(source, i0, min(nq, i0 + rows_per), dev))
                      for i0 in range(0, nq, rows_per))
        else:
            chunks = g.source_chunks(source, rows_per)
    shape = (g.tB[0].shape[1],) + tuple(s.dimension for s in reversed(st.spatial))
    acc = None
    for i0, i1, fv in chunks:
        if acc is None:
            if isinstance(fv, np.ndarray):
                acc = np.zeros(shape)
            else:                                         # device-evaluated source: contract on the device
                import torch
                acc = torch.zeros(shape, dtype=torch.float64, device=fv.device)
                ws = torch.as_tensor(ws, device=fv.device)
        if isinstance(fv, np.ndarray):
            live = np.flatnonzero(fv.reshape(i1 - i0, -1).any(axis=1))
        else:
            live = fv.reshape(i1 - i0, -1).any(dim=1).nonzero().flatten().cpu().numpy()
        if live.size == 0:
            continue
        rows = i0 + live
        tw = (g.tw[rows] * g.T).reshape((-1,) + (1,) * d)
        if not isinstance(fv, np.ndarray):
            tw = torch.as_tensor(tw, device=fv.device)
            live = torch.as_tensor(live, device=fv.device)
        vals = fv[live] * ws[None] * tw
        for l in range(d):
            vals = _mode(g.sB[l][0].T, vals, 1 + (d - 1 - l))
        acc += _mode(g.tB[0][rows].T, vals, 0)
    if acc is None:
        return np.zeros(st.num_dof)
    return acc.ravel() if isinstance(acc, np.ndarray) else acc.reshape(-1)


def window_elements(space, i):
    """bspline.py:270-277."""
    p = space.degree
    k = np.asarray(space.knots, float)
    bp = space.breakpoints
    lo, hi = k[max(i - p, 0)], k[min(i + p + 1, k.size - 1)]
    first = max(int(np.searchsorted(bp, lo, side="right")) - 1, 0)
    last = int(np.searchsorted(bp, hi, side="left")) - 1
    last = min(max(last, first), bp.size - 2)
    return first, last + 1


def _mapped_laplacian(problem, g, u):
    """div(D grad u) at the Gauss grid of a mapped geometry, pulled back with the inverse Jacobian and
    the map's Hessians (stabilization.py:273-295): D lap u = D sum_ab (J^-1 J^-T)_ab (d_ab u -
    sum_c H_abc g_c), g_c = sum_i (J^-1)_ic d_i u; with a FibreConductivity the metric is J^-1 D J^-T
    and div D adds sum_d (div D)_d g_d (FibreConductivity.diffusion_coefficients)."""
    from .geometry import is_fibre
    st, d = problem.space, g.d
    geo_data = g.mapped.geo.grid_data([r[0] for r in g.mapped.rules], order=2)
    jinv, hess = g.mapped.jinv, geo_data["hess"]
    fibre = is_fibre(problem.D)
    if fibre:
        MD, divD = problem.D.diffusion_coefficients(geo_data["jac"], hess, jinv)
    firsts = []
    for a in range(d):
        orders = [0] * d
        orders[a] = 1
        firsts.append(g.field(u, orders, 0))
    grad_eta = np.stack(firsts, axis=-1)                        # (Q_t, Q_s..., d)
    grad_phys = np.einsum("...ic,t...i->t...c", jinv, grad_eta)
    lap = np.zeros(grad_eta.shape[:-1])
    for a in range(d):
        for b in range(d):
            orders = [0] * d
            orders[a] += 1
            orders[b] += 1
            second = g.field(u, orders, 0) if max(orders) <= min(2, st.spatial[a].degree, st.spatial[b].degree) \
                else np.zeros_like(lap)
            corr = np.einsum("...c,t...c->t...", hess[..., a, b, :], grad_phys)
            metric = MD[..., a, b] if fibre else np.einsum("...k,...k->...", jinv[..., a, :], jinv[..., b, :])
            lap += metric[None] * (second - corr)
    if fibre:
        return lap + np.einsum("...d,t...d->t...", divD, grad_phys)
    return problem.D * lap


def compute_theta(problem, u, w, grid=None, device=0, lift=None):
    """Residual indicator (stabilization.py:235-339): the drop-in name runs the device indicator
    (theta.DeviceIndicator on boxes, theta.MappedDeviceIndicator on mapped geometries; ``grid`` is
    accepted for signature compatibility).  ``lift``: the indicator of the lifted field."""
    from .geometry import is_mapped
    from .theta import DeviceIndicator, MappedDeviceIndicator
    cls = MappedDeviceIndicator if is_mapped(problem.geometry) else DeviceIndicator
    ind = cls(problem, device)
    try:
        return ind.compute(u, w, lift=lift)
    finally:
        ind.close()


def host_compute_theta(problem, u, w, grid=None):
    """Host numpy restatement of compute_theta on a box or (map Hessians) a mapped geometry.  Used only
    by tests to cross-check the device kernels; no solver path calls it."""
    st = problem.space
    g = grid if grid is not None else GaussGrid(st, problem.geometry)
    d, T = g.d, g.T
    zero = [0] * d
    u_val = g.field(u, zero, 0)
    u_dtau = g.field(u, zero, 1)
    w_val = g.field(w, zero, 0)
    if g.mapped is not None:
        lap = _mapped_laplacian(problem, g, u)
    else:
        lap = np.zeros_like(u_val)
        Dv = problem.diffusion()
        for a in range(d):
            if st.spatial[a].degree < 2:
                continue
            orders = [0] * d
            orders[a] = 2
            lap += (Dv[a] / g.L[a] ** 2) * g.field(u, orders, 0)   # affine: metric diag(1/L^2), no Hessian term
    res = (problem.C_m * (u_dtau / T) - lap
           + problem.c1 * u_val * (u_val - problem.a) * (u_val - 1.0) + problem.c2 * u_val * w_val)
    if problem.source is not None:
        res = res - g.source_values(problem.source)
    absres = np.abs(res)
    denom = problem.C_m * (np.max(np.abs(u_val), initial=0.0) / T + np.max(np.abs(u_dtau), initial=0.0) / T)
    qt = st.time.degree + 1
    shape = [st.time.breakpoints.size - 1, qt]
    for l in reversed(range(d)):
        s = st.spatial[l]
        shape += [s.breakpoints.size - 1, s.degree + 1]
    emax = absres.reshape(shape)
    for ax in reversed(range(1, 2 * (d + 1), 2)):
        emax = emax.max(axis=ax)
    # windows: the reference uses full-basis time functions 0..N_t-1 (stabilization.py:307)
    out = np.stack([emax[a:b].max(axis=0) for a, b in (window_elements(st.time, c) for c in range(st.num_time))])
    for l in reversed(range(d)):
        axis = 1 + (d - 1 - l)
        s = st.spatial[l]
        moved = np.moveaxis(out, axis, 0)
        moved = np.stack([moved[a:b].max(axis=0) for a, b in (window_elements(s, i) for i in range(s.dimension))])
        out = np.moveaxis(moved, 0, axis)
    numer = out.reshape(st.num_time, st.num_space)
    if denom > 0.0:
        theta = np.minimum(numer / denom, 1.0)
    else:
        theta = np.zeros_like(numer)
        hot = numer > 1e-12 * numer.max(initial=0.0)
        if np.any(hot) and numer.max(initial=0.0) > 0.0:
            warnings.warn("residual indicator denominator vanished with a nonzero residual; "
                          "activating the stabilizer fully there", RuntimeWarning, stacklevel=2)
            theta[hot] = 1.0
    return ResidualIndicator(theta, greville(st.time)[1:], [greville(s) for s in st.spatial],
                             tuple(s.dimension for s in reversed(st.spatial)))
