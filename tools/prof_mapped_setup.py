"""cProfile of the fixed-point driver's setup phase for the mapped Spline Upwind solve (cfg-5 shape, 32^3 x 64)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_17500_b200 as mb
from paper_2311_17500_b200 import fixed_point as fp
from tools.solve_mapped import FIBRE, prolate_shell_geometry, s1_initial, s2_source
p, ne, ne_t = 3, 32, 64
st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, ne) for _ in range(3)], mb.SplineSpace.uniform(p, ne_t))
prob = mb.MonodomainProblem(prolate_shell_geometry(), st, source=s2_source(), D=FIBRE, u0=s1_initial)
cfg = mb.FixedPointConfig(stabilization="spline_upwind", linear_solver="iterative", linear_tol=1e-8, coefficient_rank=8)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pr = cProfile.Profile(); pr.enable()
    ws = fp._Workspace(prob, cfg, 0)
    torch.cuda.synchronize()
    pr.disable()
    print("rep", rep, "workspace seconds", time.perf_counter() - t0)
    if rep == 1:
        pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
    del ws
