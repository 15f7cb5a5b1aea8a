import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_17500_b200 as mb
from paper_2311_17500_b200.reaction import set_reaction
from paper_2311_17500_b200 import _lib
RM = {"c1": 0.26, "a": 0.13, "c2": 0.1}
p, ne, ne_t = 2, 64, 128
st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, ne) for _ in range(3)], mb.SplineSpace.uniform(p, ne_t))
op = mb.KroneckerOperator(st, 1.0, 1.0, 1e-3, RM)
N = st.num_dof
rng = np.random.default_rng(1)
dev = torch.device("cuda:0")
u = torch.from_numpy(rng.uniform(0, 1, N)).to(dev); w = torch.from_numpy(rng.uniform(0, 0.1, N)).to(dev)
x = torch.from_numpy(rng.uniform(-1, 1, N)).to(dev); y = torch.empty_like(x)
for kernel in (1, 0, 1, 0):
    _lib.call("mi_op_set_reaction_kernel", op.ctx.handle, kernel)
    for rep in range(3):
        set_reaction(op.ctx, st, 1.0, RM, u, w, None)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        op.apply_device(x, y); torch.cuda.synchronize(); t1 = time.perf_counter()
        op.apply_device(x, y); torch.cuda.synchronize(); t2 = time.perf_counter()
        print("kernel %d rep %d: first apply (with the c_w pass) %.1f ms, second %.1f ms" % (kernel, rep, 1e3*(t1-t0), 1e3*(t2-t1)), flush=True)
