"""Host tables for the device reaction correction M_R x (assembly.py:287-347).

The reference evaluates C_r = c1 (u - a)(u - 1) + c2 w at q = p+1 Gauss
points per element in every spatial direction (SpatialQuadratureData with
its default rule, assembly.py:146-155) and in time (TimeQuadratureData,
assembly.py:256-262, physical weights x T); the device kernel uses exactly
these points.
"""

import numpy as np

from . import _lib
from .device import dptr, host_ptr
from .spaces import basis_table, gauss_rule


_ELEMENT_TABLES = {}


def element_tables(space, q, scale):
    """(B, W): B[e, g, a] = value of function e + a at Gauss point g of element e (memoised: the
    fixed-point driver rebuilds the reaction every sweep on the same spaces; the result is read-only)."""
    key = (np.asarray(space.knots, float).tobytes(), int(space.degree), int(q), float(scale))
    hit = _ELEMENT_TABLES.get(key)
    if hit is not None:
        return hit
    bp = space.breakpoints
    ne = bp.size - 1
    x, w = gauss_rule(bp, q)
    T = basis_table(space, x, 0)
    p = space.degree
    # open uniform knots: element e carries functions e..e+p (the partition of unity checks it)
    rows = np.arange(ne * q).reshape(ne, q)
    cols = np.arange(ne)[:, None, None] + np.arange(p + 1)[None, None, :]
    B = T[rows[:, :, None], cols]
    if not np.allclose(B.sum(axis=2), 1.0):
        raise ValueError("element tables need an open knot vector with simple interior knots")
    out = (B, (w * scale).reshape(ne, q))
    for a in out:
        a.setflags(write=False)
    if len(_ELEMENT_TABLES) > 64:
        _ELEMENT_TABLES.pop(next(iter(_ELEMENT_TABLES)))
    _ELEMENT_TABLES[key] = out
    return out


def set_reaction(ctx, st, final_time, consts, u, w, lengths, time_rows=None, zslab=None):
    """``zslab=(z_lo, z_hi, hz_lo, hz_hi)``: the kernel runs on the input slab (global planes
    [z_lo - hz_lo, z_hi + hz_hi)); its z elements are those whose functions all lie there."""
    d = len(st.spatial)
    L = np.ones(d) if lengths is None else np.asarray(lengths, float)
    Bs, Ws, qs, nels = [], [], [], []
    for l, s in enumerate(st.spatial):
        B, W = element_tables(s, s.degree + 1, L[l])
        if zslab is not None and l == d - 1:
            f0 = zslab[0] - zslab[2]
            f1 = zslab[1] + zslab[3]
            B, W = B[f0:f1 - s.degree], W[f0:f1 - s.degree]   # element e carries functions e..e+p
        Bs.append(B.ravel()); Ws.append(W.ravel()); qs.append(s.degree + 1); nels.append(B.shape[0])
    B, W = element_tables(st.time, st.time.degree + 1, final_time)
    pt = st.time.degree
    nt_glob = st.time.dimension - 1
    r0, r1 = (0, nt_glob) if time_rows is None else time_rows
    # elements whose functions (full index e..e+pt, constrained row = full - 1)
    # touch the slab rows [r0, r1); local row of full function ft_local is
    # ft_local + (el0 - 1 - r0)
    el0 = max(0, r0 + 1 - pt)
    el1 = min(B.shape[0], r1 + 1)
    B, W = B[el0:el1], W[el0:el1]
    Bs.append(B.ravel()); Ws.append(W.ravel()); qs.append(pt + 1); nels.append(B.shape[0])
    Bh = np.ascontiguousarray(np.concatenate(Bs))
    Wh = np.ascontiguousarray(np.concatenate(Ws))
    qh = np.asarray(qs, dtype=np.int32)
    nh = np.asarray(nels, dtype=np.int32)
    ud = ctx.to_device(u)
    wd = ctx.to_device(w)
    ctx.bind_stream()
    _lib.call("mi_op_set_reaction", ctx.handle, dptr(ud), dptr(wd), float(consts["c1"]), float(consts["a"]),
              float(consts["c2"]), host_ptr(qh), host_ptr(nh), host_ptr(Bh), host_ptr(Wh))
    _lib.call("mi_op_set_reaction_rows", ctx.handle, int(el0 - 1 - r0))
