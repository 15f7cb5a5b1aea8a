"""Device GMRES with the reference's semantics (gmres, linalg.py:367-447).

Left-preconditioned, unrestarted, classical Gram-Schmidt with exactly one
re-orthogonalisation pass (CGS2), Givens rotations, stop when
|g_{j+1}| / beta <= tol (beta = ||P^-1 (b - A x0)||) or the new basis
vector vanishes.  The Krylov basis lives in HBM; all length-N work runs in
libmonoiga_b200 kernels (deterministic reductions).  Only the (j+1)-long
Hessenberg column and the Givens rotations are handled on the host (one
small device->host copy per iteration, needed for the stopping test).

The core loop (:func:`gmres_core`) is written against a small vector-ops
interface plus an optional ``allreduce`` hook, so the space-sharded solve
(sharded.py) runs the identical recurrence on local slabs with NCCL
allreduces of the dot products.
"""

import ctypes

import numpy as np
import scipy.linalg as sla
import torch

from . import _lib
from ._blas import single_thread_blas
from .device import dptr
from .errors import NonConvergenceError


def _write_log(path, history):
    with open(path, "w") as fh:
        fh.write("iteration,residual\n")
        for i, r in enumerate(history):
            fh.write("%d,%.17g\n" % (i, r))


class DeviceVecOps:
    """Krylov vector kernels of libmonoiga_b200 on one context's stream."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.h = ctx.handle

    def dots(self, V, k, w, out):
        """out[:k] = V[:k] @ w (local partial sums)."""
        n = w.numel()
        _lib.call("mi_dots", self.h, n, k, ctypes.c_void_p(V.data_ptr()), V.stride(0), dptr(w), dptr(out))

    def sub_comb(self, V, k, hvec, w):
        n = w.numel()
        _lib.call("mi_sub_combination", self.h, n, k, ctypes.c_void_p(V.data_ptr()), V.stride(0), dptr(hvec),
                  dptr(w))

    def sub_dots(self, V, k, h_in, w, h_out):
        """w -= V[:k]^T h_in, then h_out[:k] = V[:k] @ w (one fused pass over V)."""
        _lib.call("mi_cgs_pass", self.h, w.numel(), k, ctypes.c_void_p(V.data_ptr()), V.stride(0), dptr(h_in),
                  dptr(w), dptr(h_out))

    def sub_norm(self, V, k, h_in, w, nrm2):
        """w -= V[:k]^T h_in, then nrm2 = w . w (one fused pass over V)."""
        _lib.call("mi_cgs_norm_pass", self.h, w.numel(), k, ctypes.c_void_p(V.data_ptr()), V.stride(0),
                  dptr(h_in), dptr(w), dptr(nrm2))

    def normalize(self, src, nrm2, dst):
        _lib.call("mi_normalize", self.h, src.numel(), dptr(src), dptr(nrm2), dptr(dst))

    def comb(self, V, k, y, x0, out):
        n = out.numel()
        _lib.call("mi_combination", self.h, n, k, ctypes.c_void_p(V.data_ptr()), V.stride(0), dptr(y),
                  dptr(x0) if x0 is not None else ctypes.c_void_p(0), dptr(out))


def gmres_core(apply_A, apply_P, ops, b, x0, tol, m, allreduce=None, log_path=None, n_global=None):
    """CGS2 GMRES on (local) vectors; see module docstring.

    apply_A(src, dst), apply_P(src, dst): device applies on local vectors.
    allreduce(t): in-place sum over ranks of a small tensor (None = 1 rank).
    Returns (x_local, iterations, history).
    """
    dev = b.device
    n = b.numel()
    red = allreduce if allreduce is not None else (lambda t: None)
    tmp = torch.empty_like(b)
    if x0 is None:
        xs = torch.zeros_like(b)
        r = b
    else:
        xs = x0.clone()
        apply_A(xs, tmp)
        minus = torch.full((1,), -1.0, dtype=torch.float64, device=dev)
        r = torch.empty_like(b)
        ops.comb(tmp.view(1, -1), 1, minus, b, r)
    # The basis, the Hessenberg matrix and the dot-product scratch grow on demand (doubling, up to m + 1
    # vectors): memory follows the iterations used, not max_iter, so the reference's default
    # max_iter = n (linalg.py:381-382) costs nothing up front.  Running out of HBM raises MemoryError.
    cap = min(m, 32)
    V = torch.empty((cap + 1, n), dtype=torch.float64, device=dev)
    scal = torch.zeros(8 + 2 * (cap + 1), dtype=torch.float64, device=dev)
    nrm = scal[0:1]
    apply_P(r, V[0])
    ops.dots(V[0].view(1, -1), 1, V[0], nrm)
    red(nrm)
    beta = float(np.sqrt(nrm.item()))
    if beta == 0.0:
        if log_path is not None:
            _write_log(log_path, [0.0])
        return xs, 0, [0.0]
    ops.normalize(V[0], nrm, V[0])
    H = np.zeros((cap + 1, cap))
    cs, sn, gv = np.zeros(cap), np.zeros(cap), np.zeros(cap + 1)
    gv[0] = beta
    history = [1.0]
    k_done = None
    w = torch.empty_like(b)
    for j in range(m):
        if j + 1 >= V.shape[0]:
            new_cap = min(m, 2 * cap)
            try:
                grown = torch.empty((new_cap + 1, n), dtype=torch.float64, device=dev)
            except torch.cuda.OutOfMemoryError as exc:
                raise MemoryError("GMRES basis of %d vectors of %d DoFs does not fit in device memory "
                                  "(iteration %d; pass a smaller max_iter)" % (new_cap + 1, n, j)) from exc
            grown[:V.shape[0]].copy_(V)
            V = grown
            Hn = np.zeros((new_cap + 1, new_cap))
            Hn[:cap + 1, :cap] = H
            H = Hn
            cs, sn = np.resize(cs, new_cap), np.resize(sn, new_cap)
            gv = np.concatenate([gv, np.zeros(new_cap - cap)])
            scal = torch.zeros(8 + 2 * (new_cap + 1), dtype=torch.float64, device=dev)
            nrm = scal[0:1]
            cap = new_cap
        h1 = scal[8:8 + cap + 1]
        h2 = scal[8 + cap + 1:8 + 2 * (cap + 1)]
        apply_A(V[j], tmp)
        apply_P(tmp, w)
        k = j + 1
        # CGS2 (linalg.py:405-412); the fused passes read V once per subtraction + reduction
        ops.dots(V, k, w, h1)
        red(h1[:k])
        if hasattr(ops, "sub_dots"):
            ops.sub_dots(V, k, h1, w, h2)
        else:
            ops.sub_comb(V, k, h1, w)
            ops.dots(V, k, w, h2)
        red(h2[:k])
        if hasattr(ops, "sub_norm"):
            ops.sub_norm(V, k, h2, w, nrm)
        else:
            ops.sub_comb(V, k, h2, w)
            ops.dots(w.view(1, -1), 1, w, nrm)
        red(nrm)
        host = scal.cpu().numpy()
        hv = host[8:8 + k] + host[8 + cap + 1:8 + cap + 1 + k]
        hnorm = float(np.sqrt(host[0]))
        H[:k, j] = hv
        H[k, j] = hnorm
        for i in range(j):
            a_, b_ = H[i, j], H[i + 1, j]
            H[i, j] = cs[i] * a_ + sn[i] * b_
            H[i + 1, j] = -sn[i] * a_ + cs[i] * b_
        den = np.hypot(H[j, j], H[j + 1, j])
        if den == 0.0:
            cs[j], sn[j] = 1.0, 0.0
        else:
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
        H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
        H[j + 1, j] = 0.0
        gv[j + 1] = -sn[j] * gv[j]
        gv[j] = cs[j] * gv[j]
        rel = abs(gv[j + 1]) / beta
        history.append(float(rel))
        if rel <= tol or hnorm == 0.0:
            k_done = j + 1
            break
        ops.normalize(w, nrm, V[j + 1])
    if k_done is None:
        if log_path is not None:
            _write_log(log_path, history)
        raise NonConvergenceError("GMRES did not reach tol %.2e in %d iterations" % (tol, m),
                                  iterations=m, residuals=history)
    with single_thread_blas():
        y = sla.solve_triangular(H[:k_done, :k_done], gv[:k_done])
    yd = torch.from_numpy(np.ascontiguousarray(y)).to(dev)
    xout = torch.empty_like(b)
    ops.comb(V, k_done, yd, xs, xout)
    if log_path is not None:
        _write_log(log_path, history)
    return xout, k_done, history


def gmres(op, rhs, precond=None, tol=1e-8, max_iter=None, x0=None, log_path=None):
    """Returns ``(x, iterations, residual_history)`` like linalg.py:367-447.

    ``op`` / ``precond`` are device objects of this package (they expose
    ``apply_device``).  ``rhs`` / ``x0`` may be numpy arrays (then ``x`` is
    returned as numpy) or CUDA tensors.
    """
    if not hasattr(op, "apply_device"):
        raise TypeError("device gmres needs a device operator (KroneckerOperator of this package)")
    if precond is not None and not hasattr(precond, "apply_device"):
        raise TypeError("device gmres needs a device preconditioner")
    ctx = op.ctx
    ctx.bind_stream()
    as_numpy = not isinstance(rhs, torch.Tensor)
    b = ctx.to_device(rhs)
    n = b.numel()
    if n != op.shape[0]:
        raise ValueError("dimension mismatch: operator of size %d applied to vector of size %d"
                         % (op.shape[0], n))
    m = n if max_iter is None else int(max_iter)  # reference default (linalg.py:381-382)

    def P(src, dst):
        if precond is None:
            dst.copy_(src)
        else:
            precond.apply_device(src, dst)

    x0d = None if x0 is None else ctx.to_device(x0)
    x, it, hist = gmres_core(op.apply_device, P, DeviceVecOps(ctx), b, x0d, tol, m, log_path=log_path)
    return (x.cpu().numpy() if as_numpy else x), it, hist

