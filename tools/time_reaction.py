"""Time the reaction kernel (op_reaction profiling slot) at cfg4 size for one or
more builds of the library (ablations):

    python tools/time_reaction.py lib/libmonoiga_b200.so tools/exp/X/libmonoiga_b200.so ...

Each library runs in its own subprocess (ctypes loads one copy per process).
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(lib, ne, ne_t, reps, p=3):
    sys.path.insert(0, ROOT)
    import paper_2311_17500_b200._lib as L
    L.LIB_PATH = os.path.abspath(lib)
    import numpy as np
    import torch
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200.reaction import set_reaction
    RM = {"c1": 0.26, "a": 0.13, "c2": 0.1}
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, ne) for _ in range(3)], mb.SplineSpace.uniform(p, ne_t))
    op = mb.KroneckerOperator(st, 1.0, 1.0, 1e-3, RM)
    P = mb.FastDiagPreconditioner.build(st, 1.0, 1.0, 1e-3, 0.0, context=op.ctx)
    N = st.num_dof
    rng = np.random.default_rng(1)
    dev = torch.device("cuda:0")
    u = torch.from_numpy(rng.uniform(0, 1, N)).to(dev)
    w = torch.from_numpy(rng.uniform(0, 0.1, N)).to(dev)
    set_reaction(op.ctx, st, 1.0, RM, u, w, None)
    if os.environ.get("RX_STORE") is not None:
        from paper_2311_17500_b200 import _lib as LL
        LL.call("mi_op_set_reaction_store", op.ctx.handle, int(os.environ["RX_STORE"]))
    del u, w
    x = torch.from_numpy(rng.uniform(-1, 1, N)).to(dev)
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    for _ in range(2):
        op.apply_device(x, y)
        P.apply_device(y, z)
    torch.cuda.synchronize()
    op.ctx.read_profile(reset=True)
    op.ctx.profiling(True)
    for _ in range(reps):
        op.apply_device(x, y)
        P.apply_device(y, z)
    torch.cuda.synchronize()
    prof = op.ctx.read_profile(reset=True)
    ms = prof["op_reaction"][0] / reps
    parts = " ".join("%s=%.2f" % (k, v[0] / reps) for k, v in prof.items() if v[1])
    print("%-50s op_reaction %.2f ms  (N=%d, checksum %.12e)  [%s]" % (lib, ms, N, float(y.sum()), parts))


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    ne = int(os.environ.get("RX_NE", "96"))
    ne_t = int(os.environ.get("RX_NET", "192"))
    p = int(os.environ.get("RX_P", "3"))
    if "--one" in sys.argv:
        one(args[0], ne, ne_t, 3, p)
    else:
        for lib in args:
            subprocess.run([sys.executable, __file__, "--one", lib], check=False)
