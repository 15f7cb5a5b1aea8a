"""BASELINE cfg 5 shape on one GPU: the prolate-ellipsoid shell slab (geometry.prolate_shell_geometry,
our construction: the reference has no such geometry), p = 3.

  apply: z = P^-1 (A x) on the mapped geometry (Galerkin terms + zero-iterate reaction; M_s and K_s
         from the low-rank coefficients as Kronecker sums, or with --rank 0 by Gauss quadrature of the
         exact coefficients on the device), DoF/s and per-kernel ms;
  solve: the relaxed fixed-point solve (Galerkin, and with --su Spline Upwind: mapped SU stencils and
         the device mapped residual indicator) with the cross-field S1-S2 stimulus: S1 as initial data on
         the phi = 0 face (u0 lifting), S2 as a source pulse on the quadrant x < 0.5, z > 0 for
         0.3 <= t < 0.35 (not expressible as initial data).

Conductivity: cfg 5's fibre-aligned sigma_l = 1e-3 / sigma_t = 3e-4 (geometry.FibreConductivity, fibres
along the azimuth; an extension of the reference's scalar D) for the apply and both solves (the Spline
Upwind indicator takes div(D grad u) with the varying fibre tensor).  Coefficients: cfg 5's canonical rank <= 8 approximation
of |det J| and |det J| J^-1 D J^-T (geometry.LowRankCoefficients, --rank 8, the default); --rank 0
integrates the exact pulled-back coefficients (the reference's SpatialQuadratureData).

    python tools/solve_mapped.py --ne 64 --ne-t 256 --solve-ne 24 --solve-ne-t 64
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_17500_b200 as mb  # noqa: E402
from paper_2311_17500_b200.geometry import (FibreConductivity, MappedSpatialData,  # noqa: E402
                                            prolate_shell_geometry)

# BASELINE cfg 5 conductivity: sigma_l = 1e-3 along the fibres, sigma_t = 3e-4 across; fibres along the
# shell's azimuth (map direction 1).  An extension of the reference's scalar D (geometry.FibreConductivity).
FIBRE = FibreConductivity(1e-3, 3e-4, direction=0)

RM = {"c1": 0.26, "a": 0.13, "c2": 0.1}


def apply_rate(ne, ne_t, p, steps, rank=8):
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, ne) for _ in range(3)], mb.SplineSpace.uniform(p, ne_t))
    geo = prolate_shell_geometry()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sd = MappedSpatialData(st.spatial, geo, conductivity=FIBRE, coefficient_rank=rank or None)
    op = mb.KroneckerOperator(st, 1.0, 1.0, 1.0, RM, spatial_data=sd)
    P = mb.FastDiagPreconditioner.build(st, 1.0, 1.0, 1.0, RM["a"] * RM["c1"], spatial_data=sd, context=op.ctx)
    x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, st.num_dof)).cuda()
    y, z = torch.empty_like(x), torch.empty_like(x)
    op.apply_device(x, y)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    for _ in range(2):
        op.apply_device(x, y)
        P.apply_device(y, z)
    torch.cuda.synchronize()
    op.ctx.read_profile(reset=True)
    op.ctx.profiling(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        op.apply_device(x, y)
        P.apply_device(y, z)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    prof = {k: round(v[0] / steps, 3) for k, v in op.ctx.read_profile(reset=True).items() if v[1]}
    return {"mesh": [ne] * 3 + [ne_t], "p": p, "N": st.num_dof, "ms_per_apply": ms,
            "dof_per_s": st.num_dof / (ms * 1e-3), "kernel_ms": prof, "setup_s": setup,
            "detj_range": [float(np.abs(sd.detj).min()), float(np.abs(sd.detj).max())],
            "coefficients": coefficient_summary(sd)}


def coefficient_summary(sd):
    if sd is None or sd.lowrank is None:
        return "exact pulled-back coefficients (Gauss quadrature)"
    return {"max_rank": sd.lowrank.max_rank, "tol": sd.lowrank.tol, "fields": sd.lowrank.summary()}


def s1_initial(x):
    """S1: u0 = 1 on the phi = 0 face band (initial data, lifted as u0_h(x) b_0(t): DESIGN 7)."""
    return 1.0 * (x[:, 1] < 0.05)


def s2_source():
    """S2 ("u = 1 on one quadrant at t = 0.3") is not initial data: a source pulse on the quadrant
    x < 0.5, z > 0 for 0.3 <= t < 0.35."""
    def host(x, t):
        return 1.0 * (x[:, 0] < 0.5) * (x[:, 2] > 0.0) * (t >= 0.3) * (t < 0.35)

    def dev(x, t):
        s2 = (x[:, 0] < 0.5) & (x[:, 2] > 0.0) & (t >= 0.3) & (t < 0.35)
        return s2.to(x.dtype)

    return mb.DeviceSource(host, dev)


def solve(ne, ne_t, p, max_it, stab="off", rank=8):
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, ne) for _ in range(3)], mb.SplineSpace.uniform(p, ne_t))
    # both with cfg 5's fibre conductivity (the SU residual indicator takes div(D grad u) with the
    # fibre tensor varying along the map, FibreConductivity.diffusion_coefficients)
    prob = mb.MonodomainProblem(prolate_shell_geometry(), st, source=s2_source(), D=FIBRE, u0=s1_initial)
    cfg = mb.FixedPointConfig(stabilization=stab, linear_solver="iterative", linear_tol=1e-8, max_iterations=max_it,
                              coefficient_rank=rank or None)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = mb.fixed_point_solve(prob, cfg)
    torch.cuda.synchronize()
    return {"mesh": [ne] * 3 + [ne_t], "p": p, "N": st.num_dof, "wall_seconds": time.perf_counter() - t0,
            "sweeps": res.iterations, "converged": res.converged, "gmres_per_sweep": res.gmres_iterations,
            "avg_pcg": res.avg_pcg, "phase_seconds": {k: round(v, 3) for k, v in res.phase_seconds.items()},
            "stabilization": stab, "conductivity": "fibre 1e-3 / 3e-4",
            "stimulus": "S1 u0 on the phi=0 face (lifting) + S2 source pulse on a quadrant at t=0.3",
            "u_max": float(np.abs(res.u).max()),
            "coefficients": "canonical rank <= %d" % rank if rank else "exact"}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ne", type=int, default=64)
    ap.add_argument("--ne-t", type=int, default=256)
    ap.add_argument("--p", type=int, default=3)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--solve-ne", type=int, default=24)
    ap.add_argument("--solve-ne-t", type=int, default=64)
    ap.add_argument("--max-it", type=int, default=60)
    ap.add_argument("--su", action="store_true", help="also run the Spline Upwind solve")
    ap.add_argument("--no-apply", action="store_true")
    ap.add_argument("--rank", type=int, default=8, help="canonical rank cap of the coefficients (0: exact)")
    a = ap.parse_args()
    out = {"geometry": "prolate shell slab, quarter sector (radii 1/1/2, wall 0.2), degree-3 map, 8^3 elements"}
    if not a.no_apply:
        out["apply"] = apply_rate(a.ne, a.ne_t, a.p, a.steps, a.rank)
    if a.solve_ne > 0:
        out["solve_galerkin"] = solve(a.solve_ne, a.solve_ne_t, a.p, a.max_it, rank=a.rank)
        if a.su:
            out["solve_su"] = solve(a.solve_ne, a.solve_ne_t, a.p, a.max_it, "spline_upwind", rank=a.rank)
    print(json.dumps(out))
