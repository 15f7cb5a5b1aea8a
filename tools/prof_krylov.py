"""GMRES on the cfg-3 system (3D p=2 64^3 x 128, N = 37 M) for a fixed number of iterations, for an ncu
capture of the Krylov kernels (dots_partial / sub_reduce / dots_final / scale_div / comb):

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        -k regex:"sub_reduce|dots_partial|dots_final|scale_div|comb" python tools/prof_krylov.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_17500_b200 as mb  # noqa: E402
from bench import RM, front_indicator_np  # noqa: E402
from paper_2311_17500_b200.spaces import greville  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 24
st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(2, 64) for _ in range(3)], mb.SplineSpace.uniform(2, 128))
stab = mb.Stabilization(st, front_indicator_np(st.time_greville(), greville(st.spatial[0]), st.num_space), 0.1)
op = mb.KroneckerOperator(st, 1.0, 1.0, (1e-3, 4e-4, 4e-4), RM, stabilization=stab)
P = mb.FastDiagPreconditioner.build(st, 1.0, 1.0, (1e-3, 4e-4, 4e-4), RM["a"] * RM["c1"], context=op.ctx)
b = torch.from_numpy(np.random.default_rng(2).standard_normal(st.num_dof)).cuda()
try:
    mb.gmres(op, b, precond=P, tol=1e-30, max_iter=iters)
except mb.NonConvergenceError as exc:
    print("ran %d iterations" % exc.iterations)
torch.cuda.synchronize()
