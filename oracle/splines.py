"""B-spline spaces on [0, 1] -- oracle restatement of monoiga/bspline.py.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import numpy as np
import scipy.sparse as sp


def open_uniform_knots(p, ne):
    """bspline.py:21-28: p+1 zeros, ne-1 uniform interior knots, p+1 ones."""
    inner = np.linspace(0.0, 1.0, ne + 1)[1:-1]
    return np.hstack([np.zeros(p + 1), inner, np.ones(p + 1)])


def span_index(knots, p, x):
    """bspline.py:88-95: right-continuous span, x=1 in the last live span."""
    n = len(knots) - p - 1
    if x >= knots[n]:
        return n - 1
    return max(int(np.searchsorted(knots, x, side="right")) - 1, p)


def basis_and_derivs(knots, p, x, nd):
    """Cox-de Boor values and derivatives of the p+1 live functions at x.

    Follows bspline.py:98-147 (triangular table ``ndu`` with the knot
    differences in its lower triangle, then the derivative recurrence over
    two alternating rows).  Returns (first_index, D) with D[k, j] the k-th
    derivative of function first_index + j.
    """
    s = span_index(knots, p, x)
    tab = np.zeros((p + 1, p + 1))
    lft = np.zeros(p + 1)
    rgt = np.zeros(p + 1)
    tab[0, 0] = 1.0
    for j in range(1, p + 1):
        lft[j] = x - knots[s + 1 - j]
        rgt[j] = knots[s + j] - x
        carry = 0.0
        for r in range(j):
            tab[j, r] = rgt[r + 1] + lft[j - r]
            t = tab[r, j - 1] / tab[j, r]
            tab[r, j] = carry + rgt[r + 1] * t
            carry = lft[j - r] * t
        tab[j, j] = carry
    D = np.zeros((nd + 1, p + 1))
    D[0] = tab[:, p]
    for r in range(p + 1):
        rows = np.zeros((2, p + 1))
        cur, nxt = 0, 1
        rows[0, 0] = 1.0
        for k in range(1, nd + 1):
            acc = 0.0
            rk, pk = r - k, p - k
            if r >= k:
                rows[nxt, 0] = rows[cur, 0] / tab[pk + 1, rk]
                acc = rows[nxt, 0] * tab[rk, pk]
            lo = 1 if rk >= -1 else -rk
            hi = k - 1 if r - 1 <= pk else p - r
            for j in range(lo, hi + 1):
                rows[nxt, j] = (rows[cur, j] - rows[cur, j - 1]) / tab[pk + 1, rk + j]
                acc += rows[nxt, j] * tab[rk + j, pk]
            if r <= pk:
                rows[nxt, k] = -rows[cur, k - 1] / tab[pk + 1, r]
                acc += rows[nxt, k] * tab[r, pk]
            D[k, r] = acc
            cur, nxt = nxt, cur
    f = float(p)
    for k in range(1, nd + 1):
        D[k] *= f
        f *= p - k
    return s - p, D


class Space:
    """Univariate open-knot spline space (bspline.py:31-85, 150-284)."""

    def __init__(self, knots, p):
        self.knots = np.asarray(knots, dtype=float)
        self.degree = int(p)
        self.dimension = self.knots.size - p - 1
        self.breakpoints = np.unique(self.knots)

    @classmethod
    def uniform(cls, p, ne):
        return cls(open_uniform_knots(p, ne), p)

    @property
    def num_elements(self):
        return self.breakpoints.size - 1

    def greville(self):
        """bspline.py:221-231."""
        p = self.degree
        if p == 0:
            return 0.5 * (self.knots[:-1] + self.knots[1:])
        return np.array([self.knots[i + 1:i + p + 1].mean() for i in range(self.dimension)])

    def colloc(self, pts, order=0):
        """bspline.py:233-249: sparse (npts, dim) basis-derivative values."""
        pts = np.atleast_1d(np.asarray(pts, dtype=float))
        p = self.degree
        rows, cols, vals = [], [], []
        for m, x in enumerate(pts):
            f, D = basis_and_derivs(self.knots, p, float(x), min(order, p))
            rows.extend([m] * (p + 1))
            cols.extend(range(f, f + p + 1))
            vals.extend(D[order] if order <= p else np.zeros(p + 1))
        return sp.csr_matrix((vals, (rows, cols)), shape=(pts.size, self.dimension))

    def window_elements(self, i):
        """bspline.py:256-277: element range meeting the support extension."""
        p = self.degree
        lo = self.knots[max(i - p, 0)]
        hi = self.knots[min(i + p + 1, self.knots.size - 1)]
        bp = self.breakpoints
        a = max(int(np.searchsorted(bp, lo, side="right")) - 1, 0)
        b = int(np.searchsorted(bp, hi, side="left")) - 1
        b = min(max(b, a), self.num_elements - 1)
        return a, b + 1


class SpaceTime:
    """Space-time tensor space with the first time function dropped.

    bspline.py:311-420: coefficient layout (N_t, n_d, ..., n_1) in C order.
    """

    def __init__(self, spatial, time):
        self.spatial = tuple(spatial)
        self.time = time

    @property
    def d(self):
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

    def time_colloc(self, pts, order=0):
        """bspline.py:384-387."""
        return sp.csr_matrix(self.time.colloc(pts, order)[:, 1:])

    def time_greville(self):
        return self.time.greville()[1:]


def make_space_time(d, p, ne, ne_t, p_t=None):
    """Uniform space-time space; ``ne`` is an int or one count per direction."""
    nes = [ne] * d if np.isscalar(ne) else list(ne)
    return SpaceTime([Space.uniform(p, n) for n in nes],
                     Space.uniform(p if p_t is None else p_t, ne_t))
