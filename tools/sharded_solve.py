"""Run the sharded fixed-point driver (sharded.sharded_fixed_point_solve) under torchrun and print one
JSON line from rank 0 (sweeps, GMRES / PCG counts, increments, |u|, |w| and the solve wall time).

    torchrun --nproc-per-node G tools/sharded_solve.py --ne 6 6 8 --ne-t 8 --p 2 [--u0]

MI_DIST_BACKEND=gloo runs several ranks on fewer GPUs (host-staged collectives; functional only).
Without torchrun it runs the single-rank driver (fixed_point.fixed_point_solve) for comparison.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ne", type=int, nargs=3, default=[6, 6, 8])
    ap.add_argument("--ne-t", type=int, default=8)
    ap.add_argument("--p", type=int, default=2)
    ap.add_argument("--D", type=float, nargs="+", default=[1e-2, 4e-3, 4e-3])
    ap.add_argument("--stab", default="spline_upwind")
    ap.add_argument("--u0", action="store_true", help="initial data u0 = 1 on x < 0.2 instead of a source pulse")
    ap.add_argument("--single", action="store_true", help="single-rank driver (no torch.distributed)")
    a = ap.parse_args()
    import torch
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200.problem import BoxGeometry

    def pulse(x, t):
        return 1.0 * (x[:, 0] < 0.2) * (t < 0.1)

    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(a.p, n) for n in a.ne], mb.SplineSpace.uniform(a.p, a.ne_t))
    D = a.D[0] if len(a.D) == 1 else list(a.D)
    if a.u0:
        prob = mb.MonodomainProblem(BoxGeometry([1.0] * 3, 1.0), st, D=D, u0=lambda x: 1.0 * (x[:, 0] < 0.2))
    else:
        prob = mb.MonodomainProblem(BoxGeometry([1.0] * 3, 1.0), st, source=pulse, D=D)
    cfg = mb.FixedPointConfig(stabilization=a.stab, linear_solver="iterative")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.single or world == 1 and "RANK" not in os.environ:
        t0 = time.perf_counter()
        res = mb.fixed_point_solve(prob, cfg)
        rank = 0
    else:
        import torch.distributed as dist
        from paper_2311_17500_b200 import sharded as sh
        rank = int(os.environ["RANK"])
        local = int(os.environ.get("LOCAL_RANK", "0"))
        backend = os.environ.get("MI_DIST_BACKEND", "nccl")
        ndev = torch.cuda.device_count()
        local = local % ndev if backend == "gloo" else local
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        t0 = time.perf_counter()
        res = sh.sharded_fixed_point_solve(prob, cfg, device=local)
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"world": world, "N": st.num_dof, "sweeps": res.iterations, "gmres": res.gmres_iterations,
                          "pcg": res.pcg_iterations, "increments": res.increments,
                          "u": np.asarray(res.u).tolist(), "w": np.asarray(res.w).tolist(),
                          "seconds": time.perf_counter() - t0}))


if __name__ == "__main__":
    main()
