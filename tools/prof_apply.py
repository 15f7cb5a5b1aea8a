"""Run a few z = P^-1 (A x) applies at a given size (for ncu / nsight-style captures)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_17500_b200 as mb  # noqa: E402
from bench import RM, front_indicator_np  # noqa: E402
from paper_2311_17500_b200.spaces import greville  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=3)
ap.add_argument("--p", type=int, default=3)
ap.add_argument("--ne", type=int, default=96)
ap.add_argument("--ne-t", type=int, default=192)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--reaction", action="store_true")
a = ap.parse_args()
st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(a.p, a.ne) for _ in range(a.d)], mb.SplineSpace.uniform(a.p, a.ne_t))
theta = front_indicator_np(st.time_greville(), greville(st.spatial[0]), st.num_space)
stab = mb.Stabilization(st, theta, 0.1, 1.0)
u = w = None
if a.reaction:
    rng = np.random.default_rng(1)
    u = rng.uniform(0, 1, st.num_dof)
    w = rng.uniform(0, 0.1, st.num_dof)
op = mb.KroneckerOperator(st, 1.0, 1.0, 1e-3, RM, stabilization=stab, u=u, w=w)
P = mb.FastDiagPreconditioner.build(st, 1.0, 1.0, 1e-3, RM["a"] * RM["c1"], context=op.ctx)
x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, st.num_dof)).cuda()
y = torch.empty_like(x)
z = torch.empty_like(x)
for _ in range(a.iters):
    op.apply_device(x, y)
    P.apply_device(y, z)
torch.cuda.synchronize()
print("done", st.num_dof, float(z.norm()))
