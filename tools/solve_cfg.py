"""Run the device fixed-point driver on a BASELINE-shaped configuration and print
sweeps, iteration counts and the per-phase wall-time breakdown.

    python tools/solve_cfg.py --cfg 2          # 2D p=3, 128^2 x 256, SU every sweep
    python tools/solve_cfg.py --d 1 --p 2 --ne 64 --ne-t 64
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

# BASELINE configs 1-3.  The reference cannot take u0 != 0: each stimulus is a
# source pulse on the same region for t < 0.05.
PRESETS = {1: dict(d=1, p=2, ne=64, ne_t=64, sigma=[1e-3], stim=0.1),
           2: dict(d=2, p=3, ne=128, ne_t=256, sigma=[1e-3], stim=0.1),
           3: dict(d=3, p=2, ne=64, ne_t=128, sigma=[1e-3, 4e-4, 4e-4], stim=0.05)}

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=None)
ap.add_argument("--d", type=int, default=1)
ap.add_argument("--p", type=int, default=2)
ap.add_argument("--ne", type=int, default=64)
ap.add_argument("--ne-t", type=int, default=64)
ap.add_argument("--stab", default="spline_upwind")
ap.add_argument("--max-it", type=int, default=100)
ap.add_argument("--sigma", type=float, nargs="+", default=[1e-3])
ap.add_argument("--stim", type=float, default=0.1)
a = ap.parse_args()
if a.cfg is not None:
    for k, v in PRESETS[a.cfg].items():
        setattr(a, k, v)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2311_17500_b200 as mb  # noqa: E402
from paper_2311_17500_b200.problem import BoxGeometry  # noqa: E402


def pulse(x, t):
    """Stimulus stand-in: cfg 1 x < 0.1; cfg 2 the corner square [0, 0.1]^2;
    cfg 3 the plane x < 0.05 -- each for t < 0.05."""
    m = (x[:, 0] < a.stim).astype(float)
    if a.cfg == 2:
        m = m * (x[:, 1] < a.stim)
    return m * (t < 0.05)


st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(a.p, a.ne) for _ in range(a.d)], mb.SplineSpace.uniform(a.p, a.ne_t))
sigma = a.sigma[0] if len(a.sigma) == 1 else list(a.sigma)
prob = mb.MonodomainProblem(BoxGeometry([1.0] * a.d, 1.0), st, source=pulse, D=sigma)
cfg = mb.FixedPointConfig(stabilization=a.stab, linear_solver="iterative", linear_tol=1e-8, max_iterations=a.max_it)
t0 = time.perf_counter()
res = mb.fixed_point_solve(prob, cfg)
torch.cuda.synchronize()
out = {"cfg": a.cfg, "d": a.d, "p": a.p, "ne": a.ne, "ne_t": a.ne_t, "N": st.num_dof, "sigma": a.sigma,
       "stabilization": a.stab,
       "wall_s": time.perf_counter() - t0, "sweeps": res.iterations, "converged": res.converged,
       "gmres": res.gmres_iterations, "avg_gmres": res.avg_gmres, "avg_pcg": res.avg_pcg,
       "phase_s": {k: round(v, 3) for k, v in res.phase_seconds.items()},
       "last_increment": res.increments[-1]}
print(json.dumps(out))
