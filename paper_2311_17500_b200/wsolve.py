"""Recovery-variable solve on the device (reference solve_w_system,
linalg.py:502-547; pcg, linalg.py:450-499; KroneckerMassPreconditioner,
linalg.py:176-203).

((W_t + b d_e M_t) (x) M_s) w = g is solved as
  Y = (K_t^{-1} (x) I) G                      (one DMMA mode product), then
  every time row: PCG with M_s and the exact parametric Kronecker mass
  preconditioner, all rows advancing together (row-batched PCG with per-row
  alpha/beta, convergence test and iteration count, like calling the
  reference's pcg once per row).
"""

import numpy as np
import scipy.linalg as sla
import torch

from . import _lib
from ._blas import single_thread_blas
from .device import DeviceContext, dptr, host_ptr
from .errors import DecompositionError, NonConvergenceError
from .spaces import time_factors, univariate_factors


class RecoverySolver:
    def __init__(self, space_time, final_time, recovery_rate, equilibrium_rate, tol=1e-8, lengths=None,
                 device=0, context=None, spatial_data=None):
        """``spatial_data`` (geometry.MappedSpatialData): a mapped geometry, whose M_s (the PCG
        operator) is assembled by quadrature; the preconditioner stays the parametric Kronecker mass
        inverse (KroneckerMassPreconditioner(st.spatial), solver.py:202), as in the reference."""
        st = space_time
        self.ctx = context if context is not None else DeviceContext(st, device)
        ctx = self.ctx
        self.tol = float(tol)
        d = ctx.d
        L = np.ones(d) if lengths is None else np.asarray(lengths, float)
        Wt, Mt = time_factors(st, final_time)
        Kt = Wt + recovery_rate * equilibrium_rate * Mt
        try:
            with single_thread_blas():
                lu = sla.lu_factor(Kt)
        except sla.LinAlgError as exc:  # pragma: no cover - singular K_t
            raise DecompositionError("temporal recovery matrix is singular: %s" % exc) from exc
        with single_thread_blas():
            Kinv = np.ascontiguousarray(sla.lu_solve(lu, np.eye(Kt.shape[0])))
        nmax = max(ctx.n)
        M = np.zeros((d, nmax, nmax))
        Minv = np.zeros((d, nmax, nmax))
        for l, s in enumerate(st.spatial):
            Ml, _, _ = univariate_factors(s)
            n = Ml.shape[0]
            M[l, :n, :n] = L[l] * Ml          # M_s = kron_l L_l M_l (assembly.py:222-238)
            Minv[l, :n, :n] = np.linalg.inv(Ml)  # preconditioner: parametric masses (linalg.py:187-190)
        M, Minv = np.ascontiguousarray(M), np.ascontiguousarray(Minv)
        ctx.bind_stream()
        _lib.call("mi_ws_setup", ctx.handle, host_ptr(Kinv), host_ptr(M), host_ptr(Minv))
        self.nt, self.ns = ctx.nt, ctx.ns
        self.mass = None
        if spatial_data is not None:
            from .operator import SpatialMassOperator
            self.mass = SpatialMassOperator(st, spatial_data, device=ctx.device.index)

    def _mass_apply(self, src, dst):
        """Ap = (I (x) M_s) p for every time row."""
        if self.mass is not None:
            self.mass.apply_device(src, dst)
            self.ctx.bind_stream()
        else:
            _lib.call("mi_ws_mass", self.ctx.handle, dptr(src), dptr(dst), self.nt, 0)

    def _rowdots(self, a, b, out):
        _lib.call("mi_rowdots", self.ctx.handle, self.nt, self.ns, dptr(a), dptr(b), dptr(out))

    def solve(self, g, max_iter=None):
        """Returns (w, pcg_iterations) like solve_w_system (numpy in -> numpy out)."""
        ctx = self.ctx
        ctx.bind_stream()
        as_numpy = not isinstance(g, torch.Tensor)
        gd = ctx.to_device(g)
        nt, ns, h = self.nt, self.ns, ctx.handle
        if gd.numel() != nt * ns:
            raise ValueError("right-hand side length incompatible with factors")
        if not bool(torch.any(gd != 0).item()):
            z = torch.zeros_like(gd)
            return (z.cpu().numpy() if as_numpy else z), []
        max_iter = 10 * ns if max_iter is None else max_iter
        Y = torch.empty_like(gd)
        _lib.call("mi_ws_time", h, dptr(gd), dptr(Y))
        dev = gd.device
        rows = torch.empty(nt, dtype=torch.float64, device=dev)
        self._rowdots(Y, Y, rows)
        bnorm = np.sqrt(rows.cpu().numpy())
        iters = np.zeros(nt, dtype=np.int64)
        active = bnorm > 0.0                       # rows with b = 0: x = 0, 0 iterations
        x = torch.zeros_like(Y)
        r = Y.clone()
        z = torch.empty_like(Y)
        _lib.call("mi_ws_mass", h, dptr(r), dptr(z), nt, 1)
        p = z.clone()
        rz = torch.empty(nt, dtype=torch.float64, device=dev)
        self._rowdots(r, z, rz)
        Ap = torch.empty_like(Y)
        curv = torch.empty_like(rz)
        rr = torch.empty_like(rz)
        for it in range(1, max_iter + 1):
            if not active.any():
                break
            self._mass_apply(p, Ap)
            self._rowdots(p, Ap, curv)
            rz_h, curv_h = rz.cpu().numpy(), curv.cpu().numpy()
            if np.any(curv_h[active] <= 0.0):
                raise DecompositionError("operator is not positive definite")
            alpha = np.where(active, rz_h / np.where(active, curv_h, 1.0), 0.0)
            ad = torch.from_numpy(alpha).to(dev)
            _lib.call("mi_row_axpy", h, nt, ns, dptr(ad), 1.0, dptr(p), dptr(x))
            _lib.call("mi_row_axpy", h, nt, ns, dptr(ad), -1.0, dptr(Ap), dptr(r))
            self._rowdots(r, r, rr)
            rel = np.sqrt(rr.cpu().numpy()) / np.where(bnorm > 0, bnorm, 1.0)
            done = active & (rel <= self.tol)
            iters[done] = it
            active = active & ~done
            if not active.any():
                break
            _lib.call("mi_ws_mass", h, dptr(r), dptr(z), nt, 1)
            rz_new = torch.empty_like(rz)
            self._rowdots(r, z, rz_new)
            beta = np.where(active, rz_new.cpu().numpy() / np.where(active, rz_h, 1.0), 0.0)
            bd = torch.from_numpy(beta).to(dev)
            _lib.call("mi_row_xpby", h, nt, ns, dptr(bd), dptr(z), dptr(p))
            rz = rz_new
        else:
            if active.any():
                raise NonConvergenceError("PCG did not reach tol %.2e in %d iterations" % (self.tol, max_iter),
                                          iterations=max_iter)
        if active.any():
            raise NonConvergenceError("PCG did not reach tol %.2e in %d iterations" % (self.tol, max_iter),
                                      iterations=max_iter)
        out = x.reshape(-1)
        return (out.cpu().numpy() if as_numpy else out), [int(v) for v in iters]
