"""Per-rank device work of the space-sharded apply, measured on ONE GPU without collectives.

For a world size G and a rank r of the cfg-4 workload, builds that rank's z-slab backend and times
its local stages of one step (the z-slab operator on the input slab, the four owned-slab mode
products, the two y-slab mode products and the y-slab time stage).  The step's data movement (halo
exchange, two all-to-alls, pack/unpack copies) is NOT included: it is reported separately as
bytes per rank.  Used to size the multi-GPU design; a number printed here is
not a multi-GPU measurement.

    python tools/rank_cost.py --world 8 --rank 3
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_17500_b200 as mb  # noqa: E402
from bench import RM, front_indicator_np  # noqa: E402
from paper_2311_17500_b200 import sharded as sh  # noqa: E402
from paper_2311_17500_b200.spaces import greville  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--rank", type=int, default=1)
ap.add_argument("--ne", type=int, default=96)
ap.add_argument("--ne-t", type=int, default=192)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(3, a.ne) for _ in range(3)], mb.SplineSpace.uniform(3, a.ne_t))
theta = front_indicator_np(st.time_greville(), greville(st.spatial[0]), st.num_space)
stab = mb.Stabilization(st, theta, 0.1, 1.0)
L = sh.ZSlabLayout(st.num_time, [s.dimension for s in st.spatial], 3, a.rank, a.world)
be = sh.DeviceSlabBackend(L, st, 1.0, 1.0, 1e-3, RM, stabilization=stab)
rng = np.random.default_rng(0)
x_in = torch.from_numpy(rng.uniform(-1, 1, L.n_in)).cuda()
y = be.empty(L.n_own)
t1, t2 = be.empty(L.n_own), be.empty(L.n_own)
b1, b2 = be.empty(L.n_blk), be.empty(L.n_blk)


def step():
    be.apply_in(x_in, y)
    be.pc_mode(0, False, y, t1, L.nt * L.nz * L.n2, 1)
    be.pc_mode(1, False, t1, t2, L.nt * L.nz, L.n1)
    be.pc_mode(2, False, b1, b2, L.nt, L.ny * L.n1)
    be.pc_time_yslab(b2, L.y_lo, L.y_hi)
    be.pc_mode(2, True, b2, b1, L.nt, L.ny * L.n1)
    be.pc_mode(1, True, t2, t1, L.nt * L.nz, L.n1)
    be.pc_mode(0, True, t1, y, L.nt * L.nz * L.n2, 1)


for _ in range(2):
    step()
torch.cuda.synchronize()
for c in (be.op.ctx, be.pc.ctx):
    c.read_profile(reset=True)
    c.profiling(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    step()
e1.record()
torch.cuda.synchronize()
prof = {}
for c in (be.op.ctx, be.pc.ctx):
    for k, v in c.read_profile(reset=True).items():
        if v[1]:
            prof[k] = round(prof.get(k, 0.0) + v[0] / a.reps, 3)
print(json.dumps({"world": a.world, "rank": a.rank, "planes": L.nz, "halo": [L.h_lo, L.h_hi], "y_cols": L.ny,
                  "local_ms_per_step": e0.elapsed_time(e1) / a.reps, "kernels_ms": prof,
                  "halo_bytes": 8 * L.nt * (L.h_lo + L.h_hi) * L.plane,
                  "all_to_all_bytes_each": 8 * (L.n_own - L.nt * L.nz * L.ny * L.n1)}))
