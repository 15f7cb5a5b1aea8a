"""Per-slot kernel times of z = P^-1 (A x) at the cfg-2 shape (2D p = 3, 128^2 x 256) with SU and M_R."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2311_17500_b200 as mb
from bench import RM, front_indicator_np
from paper_2311_17500_b200.spaces import greville
p, ne, ne_t = 3, 128, 256
st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, ne) for _ in range(2)], mb.SplineSpace.uniform(p, ne_t))
rng = np.random.default_rng(1)
N = st.num_dof
theta = front_indicator_np(st.time_greville(), greville(st.spatial[0]), st.num_space)
stab = mb.Stabilization(st, theta, 0.1, 1.0)
u = rng.uniform(0, 1, N); w = rng.uniform(0, 0.1, N)
op = mb.KroneckerOperator(st, 1.0, 1.0, 1e-3, RM, stabilization=stab, u=u, w=w)
P = mb.FastDiagPreconditioner.build(st, 1.0, 1.0, 1e-3, 0.0, context=op.ctx)
x = torch.from_numpy(rng.uniform(-1, 1, N)).cuda(); y = torch.empty_like(x); z = torch.empty_like(x)
for _ in range(3):
    op.apply_device(x, y); P.apply_device(y, z)
torch.cuda.synchronize()
op.ctx.read_profile(reset=True); op.ctx.profiling(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 20
for _ in range(reps):
    op.apply_device(x, y); P.apply_device(y, z)
e1.record(); torch.cuda.synchronize()
prof = op.ctx.read_profile(reset=True)
print("N", N, "rank", stab.rank, "ms per apply %.3f" % (e0.elapsed_time(e1) / reps), {k: round(v[0] / reps, 3) for k, v in prof.items() if v[1]}, {k: v[1] // reps for k, v in prof.items() if v[1]})
