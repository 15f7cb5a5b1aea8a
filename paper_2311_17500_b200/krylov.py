"""Device GMRES with the reference's semantics (gmres, linalg.py:367-447).

Left-preconditioned, unrestarted, classical Gram-Schmidt with exactly one
re-orthogonalisation pass (CGS2), Givens rotations, stop when
|g_{j+1}| / beta <= tol (beta = ||P^-1 (b - A x0)||) or the new basis
vector vanishes.  The Krylov basis lives in HBM; all length-N work runs in
libmonoiga_b200 kernels (deterministic reductions).  Only the (j+1)-long
Hessenberg column and the Givens rotations are handled on the host (one
small device->host copy per iteration, needed for the stopping test).
"""

import ctypes

import numpy as np
import scipy.linalg as sla
import torch

from . import _lib
from .device import dptr
from .errors import NonConvergenceError


def _write_log(path, history):
    with open(path, "w") as fh:
        fh.write("iteration,residual\n")
        for i, r in enumerate(history):
            fh.write("%d,%.17g\n" % (i, r))


def default_max_iter(n, ctx, reserve_vectors=8, fraction=0.6):
    """Unrestarted GMRES keeps max_iter+1 basis vectors; the reference's
    default max_iter = n (linalg.py:381-382) is replaced by the HBM bound."""
    free, _ = torch.cuda.mem_get_info(ctx.device)
    cap = int(fraction * free // (8 * n)) - reserve_vectors
    return max(1, min(n, cap, 1000))


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
    h = ctx.handle
    as_numpy = not isinstance(rhs, torch.Tensor)
    b = ctx.to_device(rhs)
    n = b.numel()
    if n != op.shape[0]:
        raise ValueError("dimension mismatch: operator of size %d applied to vector of size %d"
                         % (op.shape[0], n))
    m = default_max_iter(n, ctx) if max_iter is None else int(max_iter)
    dev = ctx.device

    def out(t):
        return t.cpu().numpy() if as_numpy else t

    def P(src, dst):
        if precond is None:
            dst.copy_(src)
        else:
            precond.apply_device(src, dst)

    tmp = ctx.empty(n)
    scal = torch.empty(4 * (m + 2) + 8, dtype=torch.float64, device=dev)
    nrm = scal[0:1]
    if x0 is None:
        xs = torch.zeros(n, dtype=torch.float64, device=dev)
        r = b
    else:
        xs = ctx.to_device(x0).clone()
        op.apply_device(xs, tmp)
        minus = torch.full((1,), -1.0, dtype=torch.float64, device=dev)
        r = ctx.empty(n)
        _lib.call("mi_combination", h, n, 1, dptr(tmp), n, dptr(minus), dptr(b), dptr(r))
    V = torch.empty((m + 1, n), dtype=torch.float64, device=dev)
    P(r, V[0])
    _lib.call("mi_dots", h, n, 1, dptr(V[0]), n, dptr(V[0]), dptr(nrm))
    beta = float(np.sqrt(nrm.item()))
    if beta == 0.0:
        if log_path is not None:
            _write_log(log_path, [0.0])
        return out(xs), 0, [0.0]
    _lib.call("mi_normalize", h, n, dptr(V[0]), dptr(nrm), dptr(V[0]))
    H = np.zeros((m + 1, m))
    cs, sn, gv = np.zeros(m), np.zeros(m), np.zeros(m + 1)
    gv[0] = beta
    history = [1.0]
    k_done = None
    w = ctx.empty(n)
    h1 = scal[8:8 + m + 1]
    h2 = scal[8 + m + 1:8 + 2 * (m + 1)]
    Vp = V.data_ptr()
    for j in range(m):
        op.apply_device(V[j], tmp)
        P(tmp, w)
        k = j + 1
        _lib.call("mi_dots", h, n, k, ctypes.c_void_p(Vp), n, dptr(w), dptr(h1))
        _lib.call("mi_sub_combination", h, n, k, ctypes.c_void_p(Vp), n, dptr(h1), dptr(w))
        _lib.call("mi_dots", h, n, k, ctypes.c_void_p(Vp), n, dptr(w), dptr(h2))
        _lib.call("mi_sub_combination", h, n, k, ctypes.c_void_p(Vp), n, dptr(h2), dptr(w))
        _lib.call("mi_dots", h, n, 1, dptr(w), n, dptr(w), dptr(nrm))
        host = scal[:8 + 2 * (m + 1)].cpu().numpy()
        hv = host[8:8 + k] + host[8 + m + 1:8 + m + 1 + k]
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
        _lib.call("mi_normalize", h, n, dptr(w), dptr(nrm), dptr(V[j + 1]))
    if k_done is None:
        if log_path is not None:
            _write_log(log_path, history)
        raise NonConvergenceError("GMRES did not reach tol %.2e in %d iterations" % (tol, m),
                                  iterations=m, residuals=history)
    y = sla.solve_triangular(H[:k_done, :k_done], gv[:k_done])
    yd = torch.from_numpy(np.ascontiguousarray(y)).to(dev)
    xout = ctx.empty(n)
    _lib.call("mi_combination", h, n, k_done, ctypes.c_void_p(Vp), n, dptr(yd), dptr(xs), dptr(xout))
    if log_path is not None:
        _write_log(log_path, history)
    return out(xout), k_done, history
