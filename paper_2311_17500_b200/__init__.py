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
  (stabilization.py:401-489);
* :class:`RecoverySolver` -- the recovery-variable solve (solve_w_system,
  linalg.py:502-547) with row-batched device PCG;
* :func:`fixed_point_solve` with :class:`MonodomainProblem`,
  :class:`FixedPointConfig`, :class:`SolveResult`, :class:`FixedPointDiverged`
  (solver.py:58-386) for box geometries; :func:`compute_theta`
  (stabilization.py:235-339) on the host;
* :class:`ApplyStream` -- pipelined P^{-1} A over a queue of host vectors
  (copy-in / apply / copy-out overlapped on three CUDA streams).

All (d+1)-way tensor work runs in ``lib/libmonoiga_b200.so`` (C ABI in
``include/monoiga_b200.h``); there is no CPU fallback.
"""

from .errors import (ConsistencyError, DecompositionError, ExtensionError, NonConvergenceError,
                     StabilizationError)
from .problem import (BoxGeometry, DeviceSource, FixedPointConfig, FixedPointDiverged, MonodomainProblem, ResidualIndicator,
                      SolveResult, compute_theta)
from .spaces import SpaceTimeSpace, SplineSpace
from .geometry import FibreConductivity, GeometryMap, MappedSpatialData, load_geometry, save_geometry

__version__ = "0.1.0"

__all__ = [
    "DeviceSource",
    "SplineSpace", "SpaceTimeSpace", "KroneckerOperator", "FastDiagPreconditioner", "Stabilization",
    "gmres", "DeviceContext", "ConsistencyError", "DecompositionError", "ExtensionError",
    "NonConvergenceError", "StabilizationError", "BoxGeometry", "FixedPointConfig", "FixedPointDiverged",
    "MonodomainProblem", "ResidualIndicator", "SolveResult", "compute_theta", "fixed_point_solve",
    "RecoverySolver", "ApplyStream", "GeometryMap", "MappedSpatialData", "FibreConductivity", "load_geometry",
    "save_geometry",
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
    if name == "fixed_point_solve":
        from .fixed_point import fixed_point_solve
        return fixed_point_solve
    if name == "RecoverySolver":
        from .wsolve import RecoverySolver
        return RecoverySolver
    if name == "ApplyStream":
        from .stream import ApplyStream
        return ApplyStream
    if name == "DeviceContext":
        from .device import DeviceContext
        return DeviceContext
    raise AttributeError(name)
