"""Per-kernel-slot timing of z = P^-1 (A x) on the bench workload (cfg 4 with SU; env TV_NE / TV_NET /
TV_P / TV_REACTION=1 for the general iterate) for one or more builds of the library (ablations):

    python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/X.so ...

Each library runs in its own subprocess (ctypes loads one copy per process); the checksum shows the
variants compute the same result.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(lib, reps=5):
    sys.path.insert(0, ROOT)
    import paper_2311_17500_b200._lib as L
    L.LIB_PATH = os.path.abspath(lib)
    import numpy as np
    import torch
    import paper_2311_17500_b200 as mb
    from bench import RM, front_indicator_np
    from paper_2311_17500_b200.spaces import greville
    ne, ne_t, p = (int(os.environ.get(k, v)) for k, v in (("TV_NE", "96"), ("TV_NET", "192"), ("TV_P", "3")))
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, ne) for _ in range(3)], mb.SplineSpace.uniform(p, ne_t))
    stab = mb.Stabilization(st, front_indicator_np(st.time_greville(), greville(st.spatial[0]), st.num_space), 0.1)
    dev = torch.device("cuda:0")
    u = w = None
    if os.environ.get("TV_REACTION"):
        rng = np.random.default_rng(1)
        u = torch.from_numpy(rng.uniform(0, 1, st.num_dof)).to(dev)
        w = torch.from_numpy(rng.uniform(0, 0.1, st.num_dof)).to(dev)
    op = mb.KroneckerOperator(st, 1.0, 1.0, 1e-3, RM, stabilization=stab, u=u, w=w)
    P = mb.FastDiagPreconditioner.build(st, 1.0, 1.0, 1e-3, RM["a"] * RM["c1"], context=op.ctx)
    del u, w
    x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, st.num_dof)).to(dev)
    y, z = torch.empty_like(x), torch.empty_like(x)
    for _ in range(2):
        op.apply_device(x, y)
        P.apply_device(y, z)
    torch.cuda.synchronize()
    op.ctx.read_profile(reset=True)
    op.ctx.profiling(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        op.apply_device(x, y)
        P.apply_device(y, z)
    e1.record()
    torch.cuda.synchronize()
    prof = op.ctx.read_profile(reset=True)
    parts = " ".join("%s=%.2f" % (k, v[0] / reps) for k, v in prof.items() if v[1])
    print("%-44s apply %.2f ms  checksum %.15e  [%s]" % (lib, e0.elapsed_time(e1) / reps, float(z.sum()), parts),
          flush=True)


if __name__ == "__main__":
    if "--one" in sys.argv:
        one([a for a in sys.argv[1:] if not a.startswith("--")][0])
    else:
        for lib in sys.argv[1:]:
            subprocess.run([sys.executable, __file__, "--one", lib], check=False)
