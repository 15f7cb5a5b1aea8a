"""Bandwidth of the Krylov kernels (mi_dots, mi_cgs_pass, mi_cgs_norm_pass, mi_normalize) on cfg-3-sized
vectors (N = 37.1 M) for k basis vectors, for one or more library builds (CUDA events, best of 5):

    python tools/time_krylov.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/X.so ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(lib):
    sys.path.insert(0, ROOT)
    import paper_2311_17500_b200._lib as L
    L.LIB_PATH = os.path.abspath(lib)
    import torch
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200.device import DeviceContext
    from paper_2311_17500_b200.krylov import DeviceVecOps
    n = 37086984
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(2, 8)], mb.SplineSpace.uniform(2, 8))
    ops = DeviceVecOps(DeviceContext(st, 0))
    V = torch.randn(33, n, dtype=torch.float64, device="cuda")
    w = torch.randn(n, dtype=torch.float64, device="cuda")
    h = torch.randn(33, dtype=torch.float64, device="cuda") * 1e-3
    out = torch.zeros(33, dtype=torch.float64, device="cuda")
    res = []
    for k in (8, 16, 32):
        def two_pass():
            ops.sub_comb(V, k, h, w)
            ops.dots(V, k, w, out)

        for name, fn, nbytes in (("dots", lambda: ops.dots(V, k, w, out), (k + 1) * 8 * n),
                                 ("sub+dots", two_pass, (2 * k + 3) * 8 * n),
                                 ("cgs_pass", lambda: ops.sub_dots(V, k, h, w, out), (k + 2) * 8 * n),
                                 ("cgs_norm", lambda: ops.sub_norm(V, k, h, w, out), (k + 2) * 8 * n)):
            fn()
            best = 1e30
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            res.append("%s k=%d %.3f ms %.0f GB/s" % (name, k, best, nbytes / (best * 1e-3) / 1e9))
    print(lib, " | ".join(res), flush=True)


if __name__ == "__main__":
    if "--one" in sys.argv:
        one([a for a in sys.argv[1:] if not a.startswith("--")][0])
    else:
        for lib in sys.argv[1:]:
            subprocess.run([sys.executable, __file__, "--one", lib], check=False)
