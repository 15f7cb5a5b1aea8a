"""Left-preconditioned GMRES (CGS2 + Givens) -- restatement of linalg.py:367-447.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp


class NonConvergenceError(RuntimeError):
    def __init__(self, message, x=None, iterations=0, residuals=None):
        super().__init__(message)
        self.x, self.iterations = x, iterations
        self.residuals = [] if residuals is None else residuals


def _mv(op):
    """linalg.py:53-60."""
    if hasattr(op, "matvec"):
        return op.matvec
    if sp.issparse(op) or isinstance(op, np.ndarray):
        return lambda v: np.asarray(op @ v).ravel()
    return op


def _ps(pc):
    """linalg.py:63-72."""
    if pc is None:
        return lambda v: v
    if hasattr(pc, "apply"):
        return pc.apply
    if sp.issparse(pc) or isinstance(pc, np.ndarray):
        return lambda v: np.asarray(pc @ v).ravel()
    return pc


def gmres(op, rhs, precond=None, tol=1e-8, max_iter=None, x0=None):
    """linalg.py:367-447: returns (x, iterations, history)."""
    A, P = _mv(op), _ps(precond)
    b = np.asarray(rhs, float).ravel()
    n = b.size
    m = n if max_iter is None else max_iter
    if x0 is None:
        x0, r = np.zeros(n), b
    else:
        x0 = np.asarray(x0, float).ravel()
        r = b - A(x0)
    z = P(r)
    beta = np.linalg.norm(z)
    if beta == 0.0:
        return x0.copy(), 0, [0.0]
    V = [z / beta]
    H = np.zeros((m + 1, m))
    cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
    g[0] = beta
    hist = [1.0]
    k = None
    for j in range(m):
        wv = P(A(V[j]))
        Vm = np.array(V)
        h1 = Vm @ wv
        wv = wv - h1 @ Vm
        h2 = Vm @ wv
        wv = wv - h2 @ Vm
        hn = np.linalg.norm(wv)
        H[:j + 1, j] = h1 + h2
        H[j + 1, j] = hn
        for i in range(j):
            a_, b_ = H[i, j], H[i + 1, j]
            H[i, j] = cs[i] * a_ + sn[i] * b_
            H[i + 1, j] = -sn[i] * a_ + cs[i] * b_
        den = np.hypot(H[j, j], H[j + 1, j])
        cs[j], sn[j] = (1.0, 0.0) if den == 0.0 else (H[j, j] / den, H[j + 1, j] / den)
        H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        rel = abs(g[j + 1]) / beta
        hist.append(float(rel))
        if rel <= tol or hn == 0.0:
            k = j + 1
            break
        V.append(wv / hn)
    if k is None:
        raise NonConvergenceError("GMRES did not reach tol %.2e in %d iterations" % (tol, m),
                                  iterations=m, residuals=hist)
    y = sla.solve_triangular(H[:k, :k], g[:k])
    return x0 + y @ np.array(V[:k]), k, hist
