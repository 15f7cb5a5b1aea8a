"""Device operator of the potential system (drop-in for the reference's
``KroneckerOperator`` as built by ``_Workspace.operator``, solver.py:213-236).

A = C_m W_t (x) M_s + M_t (x) (sum_a sigma_a K_a + r M_s)        [Galerkin]
  + sum_r C_m s_r (sum_k S^t_{r,k}) (x) S^s_r                    [Spline Upwind]
  + M_R                                   [reaction, when the iterate != 0]

with r = c1 * a at the zero iterate (solver.py:220-223) and M_R the q=p+1
reaction mass otherwise (assembly.py:287-347).  Each Kronecker term is one
device "channel" (see csrc/op.cu).
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .device import DeviceContext, dptr, host_ptr
from .factors import hat_triple, lowrank_factorize, su_time_bands, upwind_weights
from .spaces import time_factors, to_band, univariate_factors


def _is_zero(v):
    if v is None:
        return True
    if isinstance(v, torch.Tensor):
        return not bool(torch.any(v != 0).item())
    return not np.any(v)


class Stabilization:
    """Spline Upwind data for the operator (stabilization.py:401-489).

    From the N_t x N_s indicator: upwind weights tau_k, truncated SVD at
    ``tol`` (rank R), per-rank time bands C_m s_r sum_k S^t_{r,k}, and the
    spatial factors theta_r with the 1D hat triple products that generate
    the stencils of S^s_r on the device.
    """

    def __init__(self, space_time, indicator, tol=0.1, capacitance=1.0, lengths=None):
        st = space_time
        self.tau = upwind_weights(st.time)
        self.capacitance = capacitance
        self.space_time = st
        self.lowrank = lowrank_factorize(indicator, tol)
        self.rank = self.lowrank.rank
        d = len(st.spatial)
        L = np.ones(d) if lengths is None else np.asarray(lengths, float)
        if self.rank:
            self.time_bands = su_time_bands(st, self.tau, self.lowrank, capacitance)
            self.theta = np.ascontiguousarray(self.lowrank.space_factors.T)
            nmax = max(s.dimension for s in st.spatial)
            tabs = [hat_triple(s, L[l]) for l, s in enumerate(st.spatial)]
            self.ko = tabs[0][1]
            p = st.spatial[0].degree
            H = np.zeros((d, nmax, 2 * p + 1, 2 * self.ko + 1))
            for l, (h, _) in enumerate(tabs):
                H[l, :h.shape[0]] = h
            self.H = H
        else:
            self.time_bands = np.zeros((0, st.num_time, 2 * st.time.degree + 1))


class KroneckerOperator:
    """Device operator A (see module docstring).

    ``matvec(x)`` accepts a numpy array (returns numpy; the host<->device
    copies are part of the call) or a CUDA tensor (returns a CUDA tensor,
    no host traffic).  Size mismatch raises ValueError like
    assembly.py:431-436.
    """

    def __init__(self, space_time, final_time, capacitance=1.0, diffusion=1e-4, constants=None,
                 u=None, w=None, stabilization=None, lengths=None, device=0, context=None, time_rows=None,
                 z_planes=None, spatial_data=None, lift=None, lift_in_reaction=True, iterate_is_zero=None):
        """``time_rows=(e_lo, e_hi)`` builds the operator restricted to a slab of
        constrained time rows: the time bands are the global rows e_lo..e_hi, and
        u, w (if given) are slab vectors.  ``z_planes=(z_lo, z_hi)`` (d = 3) builds
        the z-slab operator of the space-sharded solve (sharded.py): it maps an input
        slab (the owned planes plus up to p halo planes on each side, all time rows)
        to the owned planes of A x; u, w (if given) are input-slab vectors.
        ``spatial_data`` (a geometry.MappedSpatialData) selects a mapped geometry: M_s and K_s are
        then assembled by Gauss quadrature on the device (SpatialQuadratureData.mass/stiffness,
        assembly.py:197-219) and the reaction carries |det J| (assembly.py:320-326).
        ``lift`` (N_s coefficients of u0, numpy or device; the u0 lifting of DESIGN section 7, absent
        in the reference): the reaction sees the lifted iterate u0 b_0 + u, the zero-iterate switch
        needs u0 = 0 too, and ``lift_apply()`` returns the right-hand side correction A_{c,0} u0.
        ``lift_in_reaction=False`` keeps the Kronecker reaction term of the zero iterate (an operator
        that only uses that channel as a plain mass term, like the recovery right-hand side's).
        ``iterate_is_zero`` overrides the zero-iterate test (solver.py:220) with a decision taken
        elsewhere -- the sharded driver takes it over the GLOBAL iterate, not this rank's slab."""
        sd = spatial_data
        if sd is not None:
            if z_planes is not None or time_rows is not None:
                raise NotImplementedError("mapped geometries are not sharded")
            if np.atleast_1d(np.asarray(diffusion, float)).size != 1:
                raise ValueError("mapped geometries take a scalar diffusion (the reference's D)")
        st = space_time
        nt_glob = st.time.dimension - 1
        self.time_rows = (0, nt_glob) if time_rows is None else tuple(int(v) for v in time_rows)
        r0, r1 = self.time_rows
        zslab = None
        if z_planes is not None:
            n3, p_s = st.spatial[-1].dimension, st.spatial[-1].degree
            z_lo, z_hi = (int(v) for v in z_planes)
            zslab = (z_lo, z_hi, min(p_s, z_lo), min(p_s, n3 - z_hi))
        self.ctx = context if context is not None else DeviceContext(st, device, nt=r1 - r0, zslab=zslab)
        ctx = self.ctx
        self.space_time = st
        self.num_time, self.num_space = ctx.nt, ctx.ns
        consts = dict(c1=0.26, a=0.13, c2=0.1) if constants is None else dict(constants)
        d, p, pt = ctx.d, ctx.p, ctx.pt
        L = np.ones(d) if lengths is None else np.asarray(lengths, float)
        sig = np.atleast_1d(np.asarray(diffusion, float))
        sig = np.repeat(sig, d) if sig.size == 1 else sig
        if sig.size != d:
            raise ValueError("diffusion must be a scalar or one value per direction")
        has_lift = lift is not None and not _is_zero(lift)
        if has_lift and time_rows is not None:
            raise NotImplementedError("u0 lifting needs the whole time axis (not a time slab)")
        zero_iterate = (_is_zero(u) and _is_zero(w)) if iterate_is_zero is None else bool(iterate_is_zero)
        zero_iterate = zero_iterate and not (has_lift and lift_in_reaction)
        react = consts["c1"] * consts["a"] if zero_iterate else 0.0
        self.zero_iterate = zero_iterate
        stab = stabilization
        R = 0 if stab is None else stab.rank
        nchan = 2 + R
        self.nchan = nchan
        ctx.bind_stream()
        _lib.call("mi_op_setup", ctx.handle, nchan)
        # time bands: c0 = C_m W_t, c1 = M_t, SU ranks
        Wt, Mt = time_factors(st, final_time)
        bands = np.zeros((nchan, nt_glob, 2 * pt + 1))
        bands[0] = capacitance * to_band(Wt, pt)
        bands[1] = to_band(Mt, pt)
        if R:
            bands[2:] = stab.time_bands
        # slab rows: band entries reaching outside the slab multiply halo rows
        # whose results are discarded by the caller
        bands = np.ascontiguousarray(bands[:, r0:r1])
        _lib.call("mi_op_set_time_bands", ctx.handle, host_ptr(bands))
        # spatial Kronecker channels (1D tables are global in every direction)
        nmax = max(ctx.n[:-1] + [ctx.n3g])
        Mb, Kb = [], []
        for l, s in enumerate(st.spatial):
            M, K, _ = univariate_factors(s)
            Mb.append(L[l] * to_band(M, p))
            Kb.append(to_band(K, p) / L[l])

        def pack(rows):
            out = np.zeros((len(rows), d, nmax, 2 * p + 1))
            for t, row in enumerate(rows):
                for l in range(d):
                    out[t, l, :row[l].shape[0]] = row[l]
            return np.ascontiguousarray(out)

        if sd is not None:
            # c0 = M_s, c1 = D K_s (+ a c1 M_s at the zero iterate): the M_s and K_s stencils are
            # generated by quadrature on the device once per (geometry data, device) and combined here
            Ms, Ks = mapped_stencils(ctx, sd)
            _lib.call("mi_op_set_channel_stencil", ctx.handle, 0, dptr(Ms))
            c1s = float(sig[0]) * Ks
            if react != 0.0:
                c1s.add_(Ms, alpha=react)
            _lib.call("mi_op_set_channel_stencil", ctx.handle, 1, dptr(c1s))
            torch.cuda.current_stream(ctx.device).synchronize()
        else:
            c0 = np.array([1.0])
            b0 = pack([Mb])
            _lib.call("mi_op_set_kron_channel", ctx.handle, 0, 1, host_ptr(c0), host_ptr(b0))
            rows, coefs = [], []
            for a in range(d):
                rows.append([Kb[l] if l == a else Mb[l] for l in range(d)])
                coefs.append(sig[a])
            if react != 0.0:
                rows.append(list(Mb))
                coefs.append(react)
            c1 = np.asarray(coefs, float)
            b1 = pack(rows)
            _lib.call("mi_op_set_kron_channel", ctx.handle, 1, len(rows), host_ptr(c1), host_ptr(b1))
        if R and sd is not None:
            # mapped geometry: S^s_r by quadrature on the Greville-split rule, weight w |det J| theta_r
            su = mapped_su_data(sd)
            T = su.tables(p, nmax)
            ks = np.ascontiguousarray(su.kstart(nmax))
            kw = np.asarray(su.kw, dtype=np.int32)
            Qh = np.asarray(su.Q, dtype=np.int32)
            one = np.ones(1)
            for r in range(R):
                wr = np.ascontiguousarray(su.weight(stab.theta[r]))
                _lib.call("mi_op_set_quad_channel_k", ctx.handle, 2 + r, 1, host_ptr(one), host_ptr(wr), host_ptr(T),
                          host_ptr(ks), host_ptr(kw), host_ptr(Qh))
        for r in range(R if sd is None else 0):
            th = np.ascontiguousarray(stab.theta[r])
            H = np.ascontiguousarray(stab.H)
            _lib.call("mi_op_set_su_channel", ctx.handle, 2 + r, host_ptr(th), host_ptr(H), stab.ko)
        if not zero_iterate:
            from .reaction import set_reaction
            if u is None or w is None:
                zeros = ctx.empty(ctx.N_in).zero_()
                u = zeros if u is None else u
                w = zeros if w is None else w
            set_reaction(ctx, st, final_time, consts, u, w, None if sd is not None else L,
                         time_rows=self.time_rows, zslab=ctx.zslab)
            if sd is not None:
                jw = np.abs(sd.detj) if sd.lowrank is None else sd.lowrank.reconstruct("mass")
                jw = np.ascontiguousarray(jw)
                _lib.call("mi_op_set_reaction_weight", ctx.handle, host_ptr(jw))
        else:
            _lib.call("mi_op_clear_reaction", ctx.handle)    # a reused context may carry one
        self.has_lift = has_lift
        if has_lift:
            from .factors import su_time_lift
            from .spaces import time_lift_columns
            wcol, mcol = time_lift_columns(st, final_time)
            col0 = np.zeros((nchan, ctx.nt))
            col0[0] = capacitance * wcol
            col0[1] = mcol
            if R:
                col0[2:] = su_time_lift(st, stab.tau, stab.lowrank, stab.capacitance)
            self._lift = ctx.to_device(lift).contiguous()
            if self._lift.numel() != ctx.ns_in:
                raise ValueError("lifting coefficients must have one entry per spatial function (%d), got %d"
                                 % (ctx.ns_in, self._lift.numel()))
            _lib.call("mi_op_set_lift", ctx.handle, host_ptr(np.ascontiguousarray(col0)), dptr(self._lift))
        else:
            _lib.call("mi_op_set_lift", ctx.handle, None, None)
        # pack the channels for the tensor cores now; an operator on its own context drops the plain
        # stencil copy, a reused context (the fixed-point drivers rebuild one every sweep) keeps it
        _lib.call("mi_op_finalize", ctx.handle, 1 if context is None else 0)

    def lift_apply(self):
        """A_{c,0} u0: every term's lifted column applied to the lifting coefficients (device tensor,
        length N); the sweep solves A u~ = f - lift_apply()."""
        y = self.ctx.empty(self.num_time * self.num_space)
        if not self.has_lift:
            return y.zero_()
        self.ctx.bind_stream()
        _lib.call("mi_op_apply_lift", self.ctx.handle, dptr(y))
        return y

    @property
    def shape(self):
        """(owned outputs, inputs): square unless this is a z-slab operator."""
        return (self.num_time * self.num_space, self.ctx.N_in)

    def apply_device(self, x, y):
        """y = A x for contiguous fp64 CUDA tensors of length N (no checks)."""
        self.ctx.bind_stream()
        _lib.call("mi_op_apply", self.ctx.handle, dptr(x), dptr(y))

    def matvec_from_host(self, x_host, nparts=16, out=None):
        """A x for x in PINNED host memory (a CPU torch tensor): the host-to-device copy streams in
        ``nparts`` z-plane chunks while the stencil of the chunks already on the device runs
        (mi_op_apply_from_host).  Returns the device result (``out`` if given)."""
        if not (isinstance(x_host, torch.Tensor) and x_host.device.type == "cpu"):
            raise TypeError("matvec_from_host needs a CPU torch tensor (pinned for an asynchronous copy)")
        n, n_in = self.shape
        if x_host.numel() != n_in:
            raise ValueError("dimension mismatch: operator of size %d applied to vector of size %d"
                             % (n_in, x_host.numel()))
        xh = x_host.contiguous()
        if not xh.is_pinned():
            xh = xh.pin_memory()
        if getattr(self, "_xdev", None) is None or self._xdev.numel() != n_in:
            self._xdev = self.ctx.empty(n_in)
        y = self.ctx.empty(n) if out is None else out
        self.ctx.bind_stream()
        _lib.call("mi_op_apply_from_host", self.ctx.handle, ctypes.c_void_p(xh.data_ptr()), dptr(self._xdev),
                  dptr(y), int(nparts))
        self._xh_keep = xh           # the copy is asynchronous: keep the host buffer alive until reuse
        return y

    def matvec(self, x):
        n, n_in = self.shape
        size = x.numel() if isinstance(x, torch.Tensor) else np.asarray(x).size
        if size != n_in:
            raise ValueError("dimension mismatch: operator of size %d applied to vector of size %d"
                             % (n_in, size))
        xd = self.ctx.to_device(x)
        yd = self.ctx.empty(n)
        self.apply_device(xd, yd)
        if isinstance(x, torch.Tensor):
            return yd
        return yd.cpu().numpy()

    __call__ = matvec


def mapped_su_data(sd):
    """geometry.MappedSUData of a MappedSpatialData's spaces and map, built once and cached on it."""
    from .geometry import MappedSUData
    cache = sd.__dict__
    if "_su" not in cache:
        cache["_su"] = MappedSUData(sd.spaces, sd.geo)
    return cache["_su"]


def mapped_stencils(ctx, sd):
    """(M_s, K_s) stencils ((2p+1)^d x N_s device tensors) of a mapped geometry, generated once by
    mi_op_set_quad_channel (through ``ctx``'s channel 0, which the caller overwrites) and cached on
    the MappedSpatialData object per device (the reference assembles M_s, K_s once per _Workspace,
    solver.py:167-175)."""
    from .geometry import mass_terms, quad_tables, stiffness_terms
    cache = sd.__dict__.setdefault("_stencils", {})
    key = str(ctx.device)
    if key not in cache:
        p, d = ctx.p, ctx.d
        nmax = max(ctx.n[:-1] + [ctx.n3g])
        qh = np.asarray(sd.q, dtype=np.int32)
        Qh = np.asarray([r[0].size for r in sd.rules], dtype=np.int32)
        nsten = (2 * p + 1) ** d
        out = []
        for kind, terms in (("mass", mass_terms(sd)), ("stiffness", stiffness_terms(sd, 1.0))):
            if sd.lowrank is not None:
                # low-rank coefficients: a sum of Kronecker products of 1D weighted factors
                coef, bands = sd.lowrank.kron_terms(sd, kind, p, nmax)
                _lib.call("mi_op_set_kron_channel", ctx.handle, 0, len(coef), host_ptr(coef), host_ptr(bands))
            else:
                coef = np.asarray([t[0] for t in terms], float)
                theta = np.ascontiguousarray(np.stack([t[1] for t in terms]))
                T = quad_tables(sd, [t[2] for t in terms], p, nmax)
                _lib.call("mi_op_set_quad_channel", ctx.handle, 0, len(terms), host_ptr(coef), host_ptr(theta),
                          host_ptr(T), host_ptr(qh), host_ptr(Qh))
            buf = ctx.empty(nsten * ctx.ns)
            _lib.call("mi_op_get_channel_stencil", ctx.handle, 0, dptr(buf))
            out.append(buf)
        torch.cuda.current_stream(ctx.device).synchronize()
        cache[key] = tuple(out)
    return cache[key]


class SpatialMassOperator:
    """(I_t (x) M_s) x on the device for a mapped geometry: one channel, identity time band, M_s
    assembled by quadrature (the PCG operator of solve_w_system, linalg.py:502-547, whose M_s is
    SpatialQuadratureData.mass on mapped geometries, solver.py:173-175)."""

    def __init__(self, space_time, spatial_data, device=0, context=None):
        st, sd = space_time, spatial_data
        self.ctx = context if context is not None else DeviceContext(st, device)
        ctx = self.ctx
        p, pt = ctx.p, ctx.pt
        ctx.bind_stream()
        _lib.call("mi_op_setup", ctx.handle, 1)
        bands = np.zeros((1, ctx.nt, 2 * pt + 1))
        bands[0, :, pt] = 1.0
        _lib.call("mi_op_set_time_bands", ctx.handle, host_ptr(np.ascontiguousarray(bands)))
        Ms, _ = mapped_stencils(ctx, sd)
        _lib.call("mi_op_set_channel_stencil", ctx.handle, 0, dptr(Ms))
        _lib.call("mi_op_clear_reaction", ctx.handle)
        _lib.call("mi_op_finalize", ctx.handle, 1 if context is None else 0)
        torch.cuda.current_stream(ctx.device).synchronize()

    def apply_device(self, x, y):
        self.ctx.bind_stream()
        _lib.call("mi_op_apply", self.ctx.handle, dptr(x), dptr(y))

