"""Per-call end-to-end time of z = P^-1 (A x) from pinned host memory at cfg 4 (matvec_from_host with
nparts z-plane chunks, P^-1, D2H) for several nparts; CUDA events, best of 5."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_17500_b200 as mb  # noqa: E402
from bench import RM, front_indicator_np  # noqa: E402
from paper_2311_17500_b200.spaces import greville  # noqa: E402

st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(3, 96) for _ in range(3)], mb.SplineSpace.uniform(3, 192))
stab = mb.Stabilization(st, front_indicator_np(st.time_greville(), greville(st.spatial[0]), st.num_space), 0.1)
op = mb.KroneckerOperator(st, 1.0, 1.0, 1e-3, RM, stabilization=stab)
P = mb.FastDiagPreconditioner.build(st, 1.0, 1.0, 1e-3, RM["a"] * RM["c1"], context=op.ctx)
N = st.num_dof
xh = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, N)).pin_memory()
zh = torch.empty(N, dtype=torch.float64).pin_memory()
for nparts in (1, 2, 4, 8, 16):
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        zh.copy_(P.apply(op.matvec_from_host(xh, nparts=nparts)), non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print("nparts %2d: %.2f ms per call -> %.3f G DoF/s" % (nparts, best, N / (best * 1e-3) / 1e9), flush=True)
