"""Host-side spline descriptors and 1D factor tables for the device path.

Everything here is O(n_l) or O(n_l^2) setup on the host (n_l <= a few
hundred): knot vectors, B-spline tables at quadrature points, banded 1D
Gram factors.  The (d+1)-way tensors never touch this module.

Mirrors the reference descriptors ``SplineSpace`` / ``SpaceTimeSpace``
(bspline.py:150-420) closely enough that reference objects can be passed in
place of these (duck-typed: ``.knots``, ``.degree``, ``.dimension``,
``.spatial``, ``.time``).
"""

import numpy as np


def uniform_open_knots(degree, num_elements):
    """Open uniform knot vector on [0, 1] (bspline.py:21-28)."""
    if num_elements < 1:
        raise ValueError("num_elements must be >= 1")
    inner = np.arange(1, num_elements) / float(num_elements)
    return np.concatenate([np.zeros(degree + 1), inner, np.ones(degree + 1)])


class SplineSpace:
    """Univariate B-spline space over an open knot vector on [0, 1]."""

    def __init__(self, knots, degree):
        self.knots = np.ascontiguousarray(knots, dtype=float)
        self.degree = int(degree)
        self.dimension = self.knots.size - self.degree - 1
        self.breakpoints = np.unique(self.knots)

    @classmethod
    def uniform(cls, degree, num_elements):
        return cls(uniform_open_knots(degree, num_elements), degree)

    @property
    def num_elements(self):
        return self.breakpoints.size - 1

    def greville(self):
        return greville(self)


class SpaceTimeSpace:
    """Spatial tensor product x time space with the first time function removed.

    Coefficient layout (N_t, n_d, ..., n_1) in C order, direction 1 fastest
    (bspline.py:311-316, tensorops.py:1-7).
    """

    def __init__(self, spatial, time):
        self.spatial = tuple(spatial)
        if not 1 <= len(self.spatial) <= 3:
            raise ValueError("1 to 3 spatial directions are supported")
        self.time = time
        interior = np.asarray(time.knots)[time.degree + 1:-time.degree - 1]
        if interior.size and np.unique(interior, return_counts=True)[1].max() > 1:
            raise ValueError("temporal knot vector must have maximal smoothness")

    @property
    def num_spatial_dims(self):
        return len(self.spatial)

    @property
    def num_space(self):
        return int(np.prod([s.dimension for s in self.spatial]))

    @property
    def num_time(self):
        return self.time.dimension - 1

    @property
    def num_dof(self):
        return self.num_space * self.num_time

    @property
    def spatial_shape(self):
        return tuple(s.dimension for s in reversed(self.spatial))

    @property
    def coeff_shape(self):
        return (self.num_time,) + self.spatial_shape

    def time_greville(self):
        return greville(self.time)[1:]


def greville(space):
    p = space.degree
    k = np.asarray(space.knots, float)
    if p == 0:
        return 0.5 * (k[:-1] + k[1:])
    csum = np.concatenate([[0.0], np.cumsum(k)])
    n = k.size - p - 1
    i = np.arange(n)
    return (csum[i + p + 1] - csum[i + 1]) / p


_TABLES = {}
_TABLES_MAX = 512


def basis_table(space, x, order=0):
    """Dense (len(x), dimension) table of the order-th derivative of every basis (memoised: the
    fixed-point driver re-evaluates the same 1D tables every sweep; the result is read-only)."""
    u = np.asarray(space.knots, float)
    xa = np.atleast_1d(np.asarray(x, float))
    key = (u.tobytes(), int(space.degree), xa.tobytes(), int(order))
    hit = _TABLES.get(key)
    if hit is None:
        hit = _basis_table(space, xa, order)
        hit.setflags(write=False)
        if len(_TABLES) >= _TABLES_MAX:
            _TABLES.pop(next(iter(_TABLES)))
        _TABLES[key] = hit
    return hit


def _basis_table(space, x, order=0):
    """Dense (len(x), dimension) table of the order-th derivative of every basis.

    Vectorised bottom-up recursion over degrees on all points at once, with
    the derivative formula D N_{i,q} = q/(u_{i+q}-u_i) N_{i,q-1}
    - q/(u_{i+q+1}-u_{i+1}) N_{i+1,q-1}.  Intervals are half-open
    [u_i, u_{i+1}); x = 1 belongs to the last non-empty span.
    """
    u = np.asarray(space.knots, float)
    p = space.degree
    x = np.atleast_1d(np.asarray(x, float))
    m = u.size - 1
    N = np.zeros((x.size, m))
    for i in range(m):
        if u[i] < u[i + 1]:
            N[:, i] = (x >= u[i]) & (x < u[i + 1])
    last = np.nonzero(u[:-1] < u[1:])[0][-1]
    N[x >= u[-1], last] = 1.0
    if order > p:
        return np.zeros((x.size, u.size - p - 1))

    def ratio(num, den):
        out = np.zeros_like(num)
        nz = den != 0.0
        out[..., nz] = num[..., nz] / den[nz]
        return out

    tables = [N]
    for q in range(1, p + 1):
        nf = u.size - q - 1
        i = np.arange(nf)
        left = ratio((x[:, None] - u[i][None, :]), u[i + q] - u[i]) * N[:, i]
        right = ratio((u[i + q + 1][None, :] - x[:, None]), u[i + q + 1] - u[i + 1]) * N[:, i + 1]
        N = left + right
        tables.append(N)
    # derivative: differentiate `order` times starting from degree p - order
    D = tables[p - order]
    for q in range(p - order + 1, p + 1):
        nf = u.size - q - 1
        i = np.arange(nf)
        a = np.zeros(nf)
        b = np.zeros(nf)
        da = u[i + q] - u[i]
        db = u[i + q + 1] - u[i + 1]
        a[da != 0] = q / da[da != 0]
        b[db != 0] = q / db[db != 0]
        D = a[None, :] * D[:, i] - b[None, :] * D[:, i + 1]
    return D


def gauss_rule(cells, q):
    """Per-cell Gauss-Legendre nodes/weights over a partition of [0, 1]."""
    cells = np.asarray(cells, float)
    xg, wg = np.polynomial.legendre.leggauss(int(q))
    a, b = cells[:-1, None], cells[1:, None]
    h = 0.5 * (b - a)
    return (a + h * (xg + 1.0)).ravel(), (h * wg).ravel()


def cells_with(space, extra=None):
    c = space.breakpoints
    if extra is not None:
        e = np.asarray(extra, float)
        c = np.unique(np.concatenate([c, e[(e > 0.0) & (e < 1.0)]]))
    return c


def gram(space, a, b, x, w):
    Bi = basis_table(space, x, a)
    Bj = basis_table(space, x, b)
    return (Bi * w[:, None]).T @ Bj


def univariate_factors(space, q=None, weight=1.0):
    """(M, K, W) dense n x n with W[i, j] = int b'_j b_i (assembly.py:85-118)."""
    q = space.degree + 1 if q is None else q
    x, w = gauss_rule(space.breakpoints, q)
    w = w * weight
    return gram(space, 0, 0, x, w), gram(space, 1, 1, x, w), gram(space, 0, 1, x, w)


def to_band(A, p):
    """Dense n x n banded matrix -> (n, 2p+1) with band[i, k] = A[i, i-p+k]."""
    n = A.shape[0]
    band = np.zeros((n, 2 * p + 1))
    for k in range(2 * p + 1):
        off = k - p
        i = np.arange(max(0, -off), min(n, n - off))
        band[i, k] = A[i, i + off]
    resid = A.copy()
    for k in range(2 * p + 1):
        off = k - p
        i = np.arange(max(0, -off), min(n, n - off))
        resid[i, i + off] = 0.0
    if np.max(np.abs(resid), initial=0.0) > 0.0:
        raise ValueError("matrix is not banded with half-bandwidth %d" % p)
    return band


def time_factors(st, final_time):
    """(W_t, M_t): constrained time advection and T-scaled mass (assembly.py:125-134)."""
    M, _, W = univariate_factors(st.time)
    return W[1:, 1:].copy(), final_time * M[1:, 1:]


def time_lift_columns(st, final_time):
    """(W[1:, 0], T M[1:, 0]): the columns of the FULL time factors that couple the constrained rows to
    the dropped first function b_0 (the u0 lifting)."""
    M, _, W = univariate_factors(st.time)
    return W[1:, 0].copy(), final_time * M[1:, 0]


def greville_points(spaces):
    """Tensor Greville abscissae as (N_s, d) parametric points, direction 1 fastest (C order)."""
    d = len(spaces)
    g = [greville(s) for s in spaces]
    mesh = np.meshgrid(*[g[l] for l in reversed(range(d))], indexing="ij")
    return np.stack([mesh[d - 1 - l].ravel() for l in range(d)], axis=1)
