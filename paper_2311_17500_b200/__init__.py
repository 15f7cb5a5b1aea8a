"""B200-native preconditioned space-time Krylov solve (hot path of arxiv 2311.17500).

Drop-in device counterparts of the reference package ``monoiga``'s hot-path
entry points:

* :class:`KroneckerOperator` -- the potential-system operator of
  ``_Workspace.operator`` (solver.py:213-236) with ``.matvec``/``.shape``;
* :class:`FastDiagPreconditioner` -- ``.build``/``.apply``/``__call__``
  (linalg.py:206-356);
* :func:`gmres` -- same signature, return value and exceptions
  (linalg.py:367-447);
* :class:`Stabilization` -- Spline Upwind terms from an indicator
  (stabilization.py:401-489).

All (d+1)-way tensor work runs in ``lib/libmonoiga_b200.so`` (C ABI in
``include/monoiga_b200.h``); there is no CPU fallback.
"""

from .errors import (ConsistencyError, DecompositionError, ExtensionError, NonConvergenceError,
                     StabilizationError)
from .spaces import SpaceTimeSpace, SplineSpace

__version__ = "0.1.0"

__all__ = [
    "SplineSpace", "SpaceTimeSpace", "KroneckerOperator", "FastDiagPreconditioner", "Stabilization",
    "gmres", "DeviceContext", "ConsistencyError", "DecompositionError", "ExtensionError",
    "NonConvergenceError", "StabilizationError",
]


def __getattr__(name):
    # device modules import torch; keep the package importable for host-only use
    if name in ("KroneckerOperator", "Stabilization"):
        from . import operator
        return getattr(operator, name)
    if name == "FastDiagPreconditioner":
        from .precond import FastDiagPreconditioner
        return FastDiagPreconditioner
    if name == "gmres":
        from .krylov import gmres
        return gmres
    if name == "DeviceContext":
        from .device import DeviceContext
        return DeviceContext
    raise AttributeError(name)
