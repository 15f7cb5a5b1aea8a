"""Device fast-diagonalisation preconditioner (drop-in for the reference's
``FastDiagPreconditioner``, linalg.py:206-356).

It inverts the parametric surrogate
    C_m W_t (x) M_s + M_t (x) (sum_l sigma_l K_l-term + react M_s)
exactly through per-direction eigenbases and the bordered time pencil
(real 2x2-block form, factors.RealTimePencil).
"""

import numpy as np
import torch

from . import _lib
from .device import DeviceContext, dptr, host_ptr
from .factors import mapped_spatial_eigs, spatial_eigs, time_pencil


class FastDiagPreconditioner:
    """P^-1 on the device.  ``apply(r)``/``__call__`` return a real copy.

    Built with :meth:`build` (signature of linalg.py:264-273, plus
    ``lengths`` for non-unit boxes, ``device``/``context``).  ``diffusion``
    may be one conductivity per direction (anisotropic extension).
    """

    def __init__(self, space_time, eigs, pencil, capacitance, diffusion, reaction, device=0, context=None):
        st = space_time
        self.ctx = context if context is not None else DeviceContext(st, device)
        ctx = self.ctx
        d = ctx.d
        sig = np.atleast_1d(np.asarray(diffusion, float))
        sig = np.repeat(sig, d) if sig.size == 1 else sig
        self.capacitance = float(capacitance)
        self.diffusion = sig
        self.reaction = float(reaction)
        self.spatial_eigs = eigs
        self.pencil = pencil
        self.num_time, self.num_space = ctx.nt, ctx.ns
        nmax = max(ctx.n)
        U = np.zeros((d, nmax, nmax))
        lam = np.zeros((d, nmax))
        for l, (Ul, ll) in enumerate(eigs):
            n = Ul.shape[0]
            U[l, :n, :n] = Ul
            lam[l, :n] = sig[l] * ll
        diag, off, partner = pencil.coupling()
        arrs = [np.ascontiguousarray(a) for a in (U, lam, pencil.Q, diag, off, pencil.g, pencil.g_low)]
        part = np.ascontiguousarray(partner.astype(np.int32))
        ctx.bind_stream()
        _lib.call("mi_pc_setup", ctx.handle, host_ptr(arrs[0]), host_ptr(arrs[1]), self.capacitance,
                  self.reaction, host_ptr(arrs[2]), host_ptr(arrs[3]), host_ptr(arrs[4]), host_ptr(part),
                  host_ptr(arrs[5]), host_ptr(arrs[6]), float(pencil.sigma))

    @classmethod
    def build(cls, space_time, final_time, capacitance, diffusion, reaction, spatial_data=None,
              lengths=None, device=0, context=None):
        """linalg.py:264-307.  Boxes: the separable weights are the constants applied by
        factors.spatial_eigs (``spatial_data`` may be omitted).  Mapped geometries: pass a
        geometry.MappedSpatialData; the per-direction factors are weighted by the rank-one
        surrogates of |det J| and of the metric (linalg.py:228-262, 286-296)."""
        from .geometry import MappedSpatialData
        if isinstance(spatial_data, MappedSpatialData):
            eigs = mapped_spatial_eigs(spatial_data)
        else:
            eigs = spatial_eigs(space_time, lengths)
        pen = time_pencil(space_time, final_time)
        return cls(space_time, eigs, pen, capacitance, diffusion, reaction, device, context)

    @property
    def shape(self):
        n = self.num_time * self.num_space
        return (n, n)

    def apply_device(self, r, z):
        self.ctx.bind_stream()
        _lib.call("mi_pc_apply", self.ctx.handle, dptr(r), dptr(z))

    def apply(self, r):
        n = self.shape[0]
        size = r.numel() if isinstance(r, torch.Tensor) else np.asarray(r).size
        if size != n:
            raise ValueError("dimension mismatch in preconditioner application")
        rd = self.ctx.to_device(r)
        zd = self.ctx.empty(n)
        self.apply_device(rd, zd)
        if isinstance(r, torch.Tensor):
            return zd
        return zd.cpu().numpy()

    __call__ = apply
