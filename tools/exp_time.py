"""Time the operator apply with an alternative build of the library (ablations)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys, os, shutil
lib = sys.argv[1]
import paper_2311_17500_b200._lib as L
L.LIB_PATH = os.path.abspath(lib)
import numpy as np, torch
sys.argv = [sys.argv[0]]
import paper_2311_17500_b200 as mb
from bench import RM, front_indicator_np
from paper_2311_17500_b200.spaces import greville
NE, NET = int(os.environ.get('NE', 96)), int(os.environ.get('NET', 192))
DD, PP = int(os.environ.get('D', 3)), int(os.environ.get('P', 3))
NEZ = int(os.environ.get('NEZ', NE))   # last spatial direction (slab experiments)
st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(PP, NE) for _ in range(DD - 1)] + [mb.SplineSpace.uniform(PP, NEZ)], mb.SplineSpace.uniform(PP, NET))
theta = front_indicator_np(st.time_greville(), greville(st.spatial[0]), st.num_space)
stab = mb.Stabilization(st, theta, 0.1, 1.0)
op = mb.KroneckerOperator(st, 1.0, 1.0, 1e-3, RM, stabilization=stab)
x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, st.num_dof)).cuda(); y = torch.empty_like(x)
for _ in range(3): op.apply_device(x, y)
torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): op.apply_device(x, y)
e1.record(); torch.cuda.synchronize(); print(lib, "apply A ms", e0.elapsed_time(e1) / 5)
P = mb.FastDiagPreconditioner.build(st, 1.0, 1.0, 1e-3, RM["a"] * RM["c1"], context=op.ctx)
z = torch.empty_like(x)
for _ in range(3): P.apply_device(y, z)
torch.cuda.synchronize(); e0.record()
for _ in range(5): P.apply_device(y, z)
e1.record(); torch.cuda.synchronize(); print(lib, "P^-1 ms", e0.elapsed_time(e1) / 5, "checksum", float(z.double().norm()))
op.ctx.read_profile(reset=True); op.ctx.profiling(True)
for _ in range(5):
    op.apply_device(x, y); P.apply_device(y, z)
torch.cuda.synchronize()
prof = op.ctx.read_profile(reset=True); op.ctx.profiling(False)
print(lib, "N", st.num_dof, "kernels ms/apply", {k: round(v[0] / 5, 3) for k, v in prof.items() if v[1]})
