"""Spline Upwind residual indicator on the device (reference compute_theta,
stabilization.py:235-339).

``DeviceIndicator(problem).compute(u, w)`` returns the same
``ResidualIndicator`` as the reference: the strong residual

    res = C_m u_t / T - sum_l D_l u_ll + c1 u (u - a)(u - 1) + c2 u w - f

at the q = p+1 Gauss points of every space-time element (kernel
``theta_elements``, csrc/theta.cu), element maxima of |res|, the window
maxima over each basis function's support (the reference's full-basis time
windows 0..N_t-1 included, stabilization.py:307), and
theta = min(numer / denom, 1) with denom = C_m (max|u| + max|u_t|) / T.

The source is a Python callable, as in the reference; it is evaluated on the
host one chunk of time elements at a time and streamed to the device, so the
full space-time Gauss grid is never materialised.
"""

import warnings

import numpy as np
import torch

from . import _lib
from .device import DeviceContext, dptr, host_ptr
from .problem import GaussGrid, ResidualIndicator, box_of, device_capable, window_elements
from .spaces import basis_table, gauss_rule, greville


def element_tables(space, order):
    """B[e, g, a] = order-th parametric derivative of function e + a at Gauss point g (q = p+1) of
    element e (open uniform knots: element e carries functions e..e+p)."""
    bp = space.breakpoints
    ne = bp.size - 1
    p = space.degree
    q = p + 1
    x, _ = gauss_rule(bp, q)
    T = basis_table(space, x, order)
    B = np.zeros((ne, q, p + 1))
    for e in range(ne):
        B[e] = T[e * q:(e + 1) * q, e:e + p + 1]
    return B


class DeviceIndicator:
    """Per-problem device state for compute_theta (tables uploaded once)."""

    def __init__(self, problem, device=0, context=None, chunk_points=1 << 26, cache_bytes=None):
        st = problem.space
        self.problem = problem
        self.st = st
        self.d = len(st.spatial)
        self.ctx = context if context is not None else DeviceContext(st, device)
        ctx = self.ctx
        p = ctx.p
        if ctx.pt != p or p > 3:
            raise ValueError("device residual indicator needs p = p_t <= 3")
        self.L, _ = box_of(problem.geometry)
        self.T = float(problem.final_time)
        B0, B1, nel = [], [], []
        for s in st.spatial:
            B0.append(element_tables(s, 0).ravel())
            B1.append(element_tables(s, 2).ravel())
            nel.append(s.breakpoints.size - 1)
        B0.append(element_tables(st.time, 0).ravel())
        B1.append(element_tables(st.time, 1).ravel())
        nel.append(st.time.breakpoints.size - 1)
        self.nel = [int(v) for v in nel]
        b0 = np.ascontiguousarray(np.concatenate(B0))
        b1 = np.ascontiguousarray(np.concatenate(B1))
        nh = np.asarray(self.nel, dtype=np.int32)
        Lh = np.ascontiguousarray(np.asarray(self.L, float))
        Dh = np.ascontiguousarray(problem.diffusion(), dtype=float)
        _lib.call("mi_theta_setup", ctx.handle, host_ptr(nh), host_ptr(b0), host_ptr(b1), host_ptr(Lh),
                  host_ptr(Dh), self.T, float(problem.C_m), float(problem.c1), float(problem.a),
                  float(problem.c2))
        self.chunk_points = int(chunk_points)
        if cache_bytes is None:   # default: up to a quarter of the device memory free now
            cache_bytes = torch.cuda.mem_get_info(ctx.device)[0] // 4
        self.cache_bytes = int(cache_bytes)
        self._grid = None
        self._src_cache = None        # [(et0, et1, device tensor)] when the source fits cache_bytes
        # support windows (element ranges) of every function, time windows over the full basis
        self.win_t = [window_elements(st.time, c) for c in range(st.num_time)]
        self.win_s = [[window_elements(s, i) for i in range(s.dimension)] for s in st.spatial]

    def _plan(self):
        if self._grid is None:
            self._grid = GaussGrid(self.st, self.problem.geometry)
        qt = self.st.time.degree + 1
        per_el = qt * int(np.prod([x.size for x in self._grid.sx]))
        nel_t = self.nel[self.d]
        keep = per_el * nel_t * 8 <= self.cache_bytes
        return qt, per_el, max(1, self.chunk_points // per_el), keep

    def source_chunks(self, source):
        """Evaluate the source chunk by chunk (host, like the reference), yielding
        (i0, i1, values) time Gauss rows for other consumers (the load vector) while the
        device copies are kept for compute() when they fit cache_bytes."""
        qt, per_el, step, keep = self._plan()
        nel_t = self.nel[self.d]
        chunks = []
        on_device = device_capable(source)
        for et0 in range(0, nel_t, step):
            et1 = min(nel_t, et0 + step)
            if on_device:                                 # evaluated by source.torch on the GPU
                fv = self._grid.source_rows_device(source, et0 * qt, et1 * qt, self.ctx.device)
                fd = fv.reshape(-1)
            else:
                fv = self._grid.source_rows(source, et0 * qt, et1 * qt)
                fd = torch.from_numpy(np.ascontiguousarray(fv.reshape(-1))).to(self.ctx.device) if keep else None
            if keep:
                chunks.append((et0, et1, fd))
            yield et0 * qt, et1 * qt, fv
        if keep:
            self._src_cache = chunks

    def _source_chunks(self, source, nel_t):
        if self._src_cache is not None:
            yield from self._src_cache
            return
        for i0, i1, fv in self.source_chunks(source):
            qt = self.st.time.degree + 1
            fd = fv.reshape(-1) if torch.is_tensor(fv) else torch.from_numpy(np.ascontiguousarray(fv.reshape(-1)))
            yield i0 // qt, i1 // qt, fd.to(self.ctx.device)

    def _window(self, src, dst, outer, n_in, wins, inner):
        w0 = np.ascontiguousarray([a for a, _ in wins], dtype=np.int32)
        w1 = np.ascontiguousarray([b for _, b in wins], dtype=np.int32)
        _lib.call("mi_window_max", self.ctx.handle, dptr(src), dptr(dst), int(outer), int(n_in), len(wins),
                  int(inner), host_ptr(w0), host_ptr(w1))

    def compute(self, u, w, on_device=False, lift=None):
        """ResidualIndicator for the state (u, w) (numpy or device tensors of length N).  With
        ``on_device`` its values stay a CUDA tensor (the driver relaxes and factorises them there).
        ``lift`` (N_s coefficients of u0): the indicator of the lifted field u0 b_0 + u (DESIGN 7)."""
        ctx, st, d = self.ctx, self.st, self.d
        ctx.bind_stream()
        ud = ctx.to_device(u)
        wd = ctx.to_device(w)
        if ud.numel() != ctx.N or wd.numel() != ctx.N:
            raise ValueError("dimension mismatch: state of size %d for a space of size %d" % (ud.numel(), ctx.N))
        if lift is not None:
            ld = ctx.to_device(lift).contiguous()
            if ld.numel() != ctx.ns:
                raise ValueError("lifting coefficients must have one entry per spatial function")
            _lib.call("mi_theta_set_lift", ctx.handle, dptr(ld))
        else:
            _lib.call("mi_theta_set_lift", ctx.handle, None)
        nel_t = self.nel[d]
        nes = int(np.prod(self.nel[:d]))
        emax = ctx.empty(nel_t * nes)
        maxes = torch.zeros(2, dtype=torch.float64, device=ctx.device)
        source = self.problem.source
        if source is None:
            _lib.call("mi_theta_elements", ctx.handle, dptr(ud), dptr(wd), None, 0, nel_t, dptr(emax),
                      dptr(maxes))
        else:
            # the source does not change between sweeps: its Gauss values stay on the device when
            # they fit cache_bytes, otherwise they are re-evaluated and streamed chunk by chunk
            for et0, et1, fd in self._source_chunks(source, nel_t):
                _lib.call("mi_theta_elements", ctx.handle, dptr(ud), dptr(wd), dptr(fd), et0, et1, dptr(emax),
                          dptr(maxes))
        return self._finish(emax, maxes, on_device)

    def _finish(self, emax, maxes, on_device):
        """Window maxima of the element maxima and the clamped ratio (stabilization.py:297-339)."""
        ctx, st, d = self.ctx, self.st, self.d
        nel_t = self.nel[d]
        nes = int(np.prod(self.nel[:d]))
        umax, utmax = (float(v) for v in maxes.cpu().numpy())
        denom = float(self.problem.C_m) * (umax / self.T + utmax / self.T)
        # window maxima: time (over elements -> functions), then x, y, z
        nt = st.num_time
        cur = ctx.empty(nt * nes)
        self._window(emax, cur, 1, nel_t, self.win_t, nes)
        del emax
        shape = [nt] + [self.nel[l] for l in reversed(range(d))]    # (nt, E_d, ..., E_1)
        for l in range(d):
            axis = d - l                                 # position of direction l in `shape`
            outer = int(np.prod(shape[:axis]))
            inner = int(np.prod(shape[axis + 1:]))
            n_out = st.spatial[l].dimension
            nxt = ctx.empty(outer * n_out * inner)
            self._window(cur, nxt, outer, shape[axis], self.win_s[l], inner)
            shape[axis] = n_out
            cur = nxt
        numer = cur
        if denom > 0.0:
            theta = ctx.empty(numer.numel())
            _lib.call("mi_theta_ratio", ctx.handle, dptr(numer), dptr(theta), int(numer.numel()), denom)
            values = theta.view(nt, st.num_space) if on_device else theta.cpu().numpy().reshape(nt, st.num_space)
        else:
            # stabilization.py:317-333 (zero denominator)
            nh = numer.cpu().numpy().reshape(nt, st.num_space)
            values = np.zeros_like(nh)
            top = nh.max(initial=0.0)
            hot = nh > 1e-12 * top
            if np.any(hot) and top > 0.0:
                warnings.warn("residual indicator denominator vanished with a nonzero residual; "
                              "activating the stabilizer fully there", RuntimeWarning, stacklevel=2)
                values[hot] = 1.0
        return ResidualIndicator(values, greville(st.time)[1:], [greville(s) for s in st.spatial],
                                 tuple(s.dimension for s in reversed(st.spatial)))

    def close(self):
        self.ctx.close()


class MappedDeviceIndicator(DeviceIndicator):
    """compute_theta on a mapped geometry (stabilization.py:235-339 with the pulled-back Laplacian,
    273-295).  Per chunk of time elements the Gauss-point fields u, u_tau, w, the first and second
    parametric derivatives of u are interpolated by tensor mode products with the 1D basis tables
    (plain dense GEMMs: cuBLAS through torch.tensordot), then ``mapped_residual_kernel``
    (csrc/theta.cu) forms the residual with the per-point metric / Hessian coefficients and the
    Rogers-McCulloch current and reduces it to element maxima; the window maxima and the ratio
    are the box path's kernels."""

    def __init__(self, problem, device=0, context=None, grid=None, chunk_points=1 << 24, cache_bytes=None):
        st = problem.space
        self.problem, self.st, self.d = problem, st, len(st.spatial)
        self.ctx = context if context is not None else DeviceContext(st, device)
        self.T = float(problem.final_time)
        self._grid = grid if grid is not None else GaussGrid(st, problem.geometry)
        g, d = self._grid, self.d
        sd = g.mapped
        if sd is None:
            raise ValueError("MappedDeviceIndicator needs a mapped geometry")
        dev = self.ctx.device
        self.tB = [torch.tensor(np.asarray(t), device=dev) for t in g.tB]
        self.tB0 = [torch.tensor(np.asarray(t), device=dev) for t in g.tB0]
        self.sB = [[torch.tensor(np.asarray(t), device=dev) for t in tl] for tl in g.sB]
        # per spatial Gauss point: cg_i = -sum_ab m_ab sum_c H_abc (J^-1)_ic, cm_ab = m_ab (x2 off-diagonal)
        gdat = sd.geo.grid_data([r[0] for r in sd.rules], order=2)
        # (on the device: per-point 3 x 3 x 3 contractions over every spatial Gauss point)
        from .geometry import is_fibre
        hess = torch.as_tensor(np.ascontiguousarray(gdat["hess"]), device=dev)
        jinv = torch.as_tensor(np.ascontiguousarray(sd.jinv), device=dev)
        hj = torch.einsum("...abc,...ic->...abi", hess, jinv)
        if is_fibre(problem.D):
            # div(D grad u) with the fibre tensor: the metric J^-1 D J^-T and the first-order term of div D
            jac = torch.as_tensor(np.ascontiguousarray(gdat["jac"]), device=dev)
            metric, divD = problem.D.diffusion_coefficients(jac, hess, jinv)
            cg = -torch.einsum("...ab,...abi->...i", metric, hj) + torch.einsum("...d,...id->...i", divD, jinv)
            self.diff = 1.0
        else:
            metric = torch.einsum("...ak,...bk->...ab", jinv, jinv)
            cg = -torch.einsum("...ab,...abi->...i", metric, hj)
            self.diff = float(problem.D)
        self.pairs = [(a, a) for a in range(d)] + [(a, b) for a in range(d) for b in range(a + 1, d)]
        coef = [cg[..., i] for i in range(d)]
        coef += [metric[..., a, b] * (1.0 if a == b else 2.0) for a, b in self.pairs]
        self.coef = torch.stack([c.reshape(-1) for c in coef]).contiguous()
        del hess, jinv, hj, metric, cg
        self.G = np.asarray([x.size for x in g.sx], dtype=np.int32)
        self.q = st.spatial[0].degree + 1
        if any(s.degree + 1 != self.q for s in st.spatial):
            raise ValueError("mapped residual indicator: equal spatial degrees required")
        self.nel = [s.breakpoints.size - 1 for s in st.spatial] + [st.time.breakpoints.size - 1]
        self.chunk_points = int(chunk_points)
        if cache_bytes is None:
            cache_bytes = torch.cuda.mem_get_info(dev)[0] // 8
        self.cache_bytes = int(cache_bytes)
        self._src_cache = None
        self.win_t = [window_elements(st.time, c) for c in range(st.num_time)]
        self.win_s = [[window_elements(s, i) for i in range(s.dimension)] for s in st.spatial]

    def _fields(self, U, W, et0, et1, lift=None):
        """(3 + d + d(d+1)/2, rows, G_s) Gauss-point fields of time elements [et0, et1); ``lift`` adds
        u0 b_0 to u (the dropped time function's column of the full time tables)."""
        st, d = self.st, self.d
        qt = st.time.degree + 1
        r0, r1 = et0 * qt, et1 * qt
        shape = tuple(s.dimension for s in reversed(st.spatial))
        memo = {}

        def spatial(X, key, orders):
            out = X
            for l in range(d):
                k = key + tuple(orders[:l + 1])
                if k not in memo:
                    o = orders[l]
                    if o >= len(self.sB[l]):                # derivative order above the degree: zero
                        memo[k] = None
                    elif out is None:
                        memo[k] = None
                    else:
                        ax = 1 + (d - 1 - l)
                        memo[k] = torch.movedim(torch.tensordot(self.sB[l][o], out, dims=([1], [ax])), 0, ax)
                out = memo[k]
            return out

        Ut = self.tB[0][r0:r1] @ U
        Utt = self.tB[1][r0:r1] @ U
        if lift is not None:
            Ut = Ut + torch.outer(self.tB0[0][r0:r1], lift)
            Utt = Utt + torch.outer(self.tB0[1][r0:r1], lift)
        Ut = Ut.reshape((r1 - r0,) + shape)
        Utt = Utt.reshape((r1 - r0,) + shape)
        Wt = (self.tB[0][r0:r1] @ W).reshape((r1 - r0,) + shape)
        zero = [0] * d
        outs = [spatial(Ut, ("u",), zero), spatial(Utt, ("ut",), zero), spatial(Wt, ("w",), zero)]
        for i in range(d):
            o = [0] * d
            o[i] = 1
            outs.append(spatial(Ut, ("u",), o))
        for a, b in self.pairs:
            o = [0] * d
            o[a] += 1
            o[b] += 1
            outs.append(spatial(Ut, ("u",), o))
        ref = outs[0]
        return torch.stack([v.reshape(r1 - r0, -1) if v is not None else torch.zeros_like(ref).reshape(r1 - r0, -1)
                            for v in outs]).contiguous()

    def compute(self, u, w, on_device=False, lift=None):
        ctx, st, d = self.ctx, self.st, self.d
        ctx.bind_stream()
        ud, wd = ctx.to_device(u), ctx.to_device(w)
        ld = None if lift is None else ctx.to_device(lift).reshape(-1)
        if ud.numel() != ctx.N or wd.numel() != ctx.N:
            raise ValueError("dimension mismatch: state of size %d for a space of size %d" % (ud.numel(), ctx.N))
        U, W = ud.view(st.num_time, -1), wd.view(st.num_time, -1)
        nel_t = self.nel[d]
        emax = torch.zeros(nel_t * int(np.prod(self.nel[:d])), dtype=torch.float64, device=ctx.device)
        maxes = torch.zeros(2, dtype=torch.float64, device=ctx.device)
        qt = st.time.degree + 1
        nel = np.asarray(self.nel[:d], dtype=np.int32)
        pr = self.problem
        source = pr.source
        if source is not None:
            chunks = self._source_chunks(source, nel_t)
        else:
            step = max(1, self.chunk_points // (qt * int(np.prod(self.G))))
            chunks = ((e0, min(nel_t, e0 + step), None) for e0 in range(0, nel_t, step))
        for et0, et1, fd in chunks:
            F = self._fields(U, W, et0, et1, ld)
            _lib.call("mi_theta_mapped_elements", ctx.handle, dptr(F), dptr(self.coef),
                      dptr(fd) if fd is not None else None, int(et0), int(et1), host_ptr(self.G), self.q, qt,
                      host_ptr(nel), self.diff, float(pr.C_m) / self.T, float(pr.c1), float(pr.a), float(pr.c2),
                      dptr(emax), dptr(maxes))
            del F
        return self._finish(emax, maxes, on_device)
