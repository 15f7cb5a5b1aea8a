"""Host profile of a WARM BASELINE cfg-1 fixed-point solve (1D p=2 64x64, SU, u0 lifting): the solve runs
once to load the library and contexts, then again under cProfile; prints the top entries."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_17500_b200 as mb  # noqa: E402
from paper_2311_17500_b200.problem import BoxGeometry  # noqa: E402

st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(2, 64)], mb.SplineSpace.uniform(2, 64))
prob = mb.MonodomainProblem(BoxGeometry([1.0], 1.0), st, D=1e-3, u0=lambda x: 1.0 * (x[:, 0] < 0.1))
cfg = mb.FixedPointConfig(stabilization="spline_upwind", linear_solver="iterative")
mb.fixed_point_solve(prob, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = mb.fixed_point_solve(prob, cfg)
print("warm solve %.3f s, %d sweeps, phases %s" % (time.perf_counter() - t0, res.iterations, res.phase_seconds))
pr = cProfile.Profile()
pr.enable()
mb.fixed_point_solve(prob, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
