"""Run small dense LAPACK calls on one BLAS thread.

The host setup calls LAPACK on matrices of a few hundred rows at most (1D eigenproblems, the time
pencil, an N_t x N_s indicator SVD, the Hessenberg triangular solve).  A many-threaded OpenBLAS spends
far longer waking its pool than computing these: on a 16-core GPU host a 65 x 66 SVD took 28 ms inside
the fixed-point driver against ~1 ms on one thread.  threadpoolctl is optional; without it nothing is
limited.
"""


class single_thread_blas:
    """Small dense LAPACK calls (N_t x N_s indicators of small problems, the N_t x N_t pencil) run on one
    BLAS thread: a many-threaded OpenBLAS spends far longer waking its pool than computing them
    (measured 28 ms per 65 x 66 SVD on a 16-core GPU host inside the fixed-point driver)."""

    def __init__(self, on=True):
        self.on = on
        self.ctx = None

    def __enter__(self):
        if self.on:
            ctl = _controller()
            if ctl is not None:
                try:
                    self.ctx = ctl.limit(limits=1, user_api="blas")
                    self.ctx.__enter__()
                except Exception:
                    self.ctx = None
        return self

    def __exit__(self, *exc):
        if self.ctx is not None:
            self.ctx.__exit__(*exc)
        return False


_CONTROLLER = []


def _controller():
    """One threadpoolctl controller per process (building one scans every loaded library: ~1 ms)."""
    if not _CONTROLLER:
        try:
            from threadpoolctl import ThreadpoolController
            _CONTROLLER.append(ThreadpoolController())
        except Exception:      # threadpoolctl is optional: then nothing is limited
            _CONTROLLER.append(None)
    return _CONTROLLER[0]
