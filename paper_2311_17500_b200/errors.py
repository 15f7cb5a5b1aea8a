"""Exceptions with the reference's names and payloads (linalg.py:32-50,
stabilization.py:33-35, solver.py:58-63)."""


class DecompositionError(RuntimeError):
    """A matrix decomposition failed or is unreliable."""


class ConsistencyError(RuntimeError):
    """A numerical consistency check failed."""


class StabilizationError(RuntimeError):
    """The Spline Upwind stabiliser cannot be constructed reliably."""


class NonConvergenceError(RuntimeError):
    """Iterative solver failed to reach the tolerance (carries x, iterations, residuals)."""

    def __init__(self, message, x=None, iterations=0, residuals=None):
        super().__init__(message)
        self.x = x
        self.iterations = iterations
        self.residuals = residuals if residuals is not None else []


class ExtensionError(RuntimeError):
    """The CUDA library is missing or a device call failed (no CPU fallback)."""
