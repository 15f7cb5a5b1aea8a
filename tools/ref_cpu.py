#!/usr/bin/env python
"""Time the UNMODIFIED reference (monoiga, installed under baseline/_ref) on the host CPU of a GPU box.

Writes profiles/r02_ref_cpu.json, which bench.py quotes as ``reference_full_size`` next to its own
numbers.  Run on the B200 box (the reference is pure Python, so it is the host's cores that count):

    python tools/ref_cpu.py [--skip-gmres]

Measured (BASELINE.md section 2 / SURVEY 8d, best of 2 unless stated):

* ``apply_cfg4_separable``: the full-size cfg-4 operator the reference can assemble (Galerkin +
  zero-iterate reaction, no SU: its SU assembly does not fit) -- KroneckerOperator.matvec and
  FastDiagPreconditioner.apply at N = 188 M, with the assembly / build times;
* ``apply_su_<mesh>``: the workload operator WITH the Spline Upwind terms (front indicator, tol 0.1)
  at the largest 3D p=3 meshes whose SU assembly finishes in minutes;
* ``gmres_cfg2``: ``gmres(op, rhs, precond=P, tol=1e-8, max_iter=300)`` on the cfg-2 sweep-1 system
  (Galerkin + zero-iterate reaction + SU, N = 4.4 M, load vector of the corner-square pulse) -- the
  same solve bench.py
  times on the GPU as ``gmres_cfg2``;
* ``fixed_point_cfg1``: ``fixed_point_solve`` with Spline Upwind and ``linear_solver="iterative"``
  at cfg 1 (1D p=2 64x64), driven by the source pulse 1[x<0.1] 1[t<0.05] (the reference has no u0).

Every entry records the host core count and the OpenBLAS thread setting.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

RM = {"c1": 0.26, "a": 0.13, "c2": 0.1}


def front(st):
    ns = st.num_space
    g1 = st.spatial[0].greville()
    gs = np.tile(g1, ns // g1.size)
    gt = st.time_greville()
    return np.clip(np.exp(-(((gs[None, :] - 0.2 - 0.5 * gt[:, None]) / 0.08) ** 2)), 0, 1)


def system(d, p, ne, ne_t, D, su):
    from monoiga.assembly import KroneckerOperator, SpatialQuadratureData, spatial_operators, time_matrices
    from monoiga.bspline import SplineSpace, SpaceTimeSpace
    from monoiga.geometry import builtin_geometry
    from monoiga.linalg import FastDiagPreconditioner
    from monoiga.stabilization import ResidualIndicator, assemble_stabilization, compute_tau, lowrank_factorize
    t0 = time.perf_counter()
    st = SpaceTimeSpace([SplineSpace.uniform(p, ne) for _ in range(d)], SplineSpace.uniform(p, ne_t))
    geo = builtin_geometry({1: "unit_interval", 2: "unit_square", 3: "unit_cube"}[d], final_time=1.0)
    W_t, M_t = time_matrices(st, 1.0)
    M_s, K_s = spatial_operators(st.spatial, geo)
    react = RM["a"] * RM["c1"]
    terms = [(1.0, W_t, M_s), (D, M_t, K_s), (react, M_t, M_s)]
    t1 = time.perf_counter()
    rank = 0
    if su:
        ind = ResidualIndicator(front(st), st.time_greville(), [s.greville() for s in st.spatial], st.spatial_shape)
        lr = lowrank_factorize(ind, 0.1)
        rank = lr.rank
        terms += assemble_stabilization(compute_tau(st.time), lr, st, geo, 1.0).terms()
    t2 = time.perf_counter()
    op = KroneckerOperator(st.num_time, st.num_space, terms)
    P = FastDiagPreconditioner.build(st, 1.0, 1.0, D, react, spatial_data=SpatialQuadratureData(st.spatial, geo))
    t3 = time.perf_counter()
    return st, op, P, {"N": st.num_dof, "su_rank": rank, "assembly_s": t1 - t0, "su_assembly_s": t2 - t1,
                       "pc_build_s": t3 - t2}


def time_apply(d, p, ne, ne_t, D, su, reps=2):
    st, op, P, rec = system(d, p, ne, ne_t, D, su)
    x = np.random.default_rng(0).uniform(-1, 1, st.num_dof)
    best_m = best_p = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        y = op.matvec(x)
        t1 = time.perf_counter()
        P.apply(y)
        t2 = time.perf_counter()
        best_m, best_p = min(best_m, t1 - t0), min(best_p, t2 - t1)
    rec.update(mesh=[ne] * d + [ne_t], d=d, p=p, matvec_s=best_m, pc_apply_s=best_p,
               dof_per_s=st.num_dof / (best_m + best_p))
    return rec


def gmres_cfg2():
    from monoiga.assembly import rhs_vectors
    from monoiga.geometry import builtin_geometry
    from monoiga.linalg import gmres

    def corner_pulse(x, t):
        return 1.0 * (x[:, 0] < 0.1) * (x[:, 1] < 0.1) * (t < 0.05)

    st, op, P, rec = system(2, 3, 128, 256, 1e-3, True)
    rhs, _ = rhs_vectors(st, builtin_geometry("unit_square", final_time=1.0), corner_pulse,
                         np.zeros(st.num_dof), 0.013)
    t0 = time.perf_counter()
    _, it, hist = gmres(op, rhs, precond=P, tol=1e-8, max_iter=300)
    rec.update(seconds=time.perf_counter() - t0, iterations=it, final_rel_residual=hist[-1],
               system="cfg2 sweep-1 system: Galerkin + zero-iterate reaction + SU (front indicator, tol 0.1), "
                      "rhs = load vector of the corner pulse 1[x<0.1, y<0.1] 1[t<0.05], tol 1e-8, max_iter 300")
    return rec


def fixed_point_cfg1():
    from monoiga.bspline import SplineSpace, SpaceTimeSpace
    from monoiga.geometry import builtin_geometry
    from monoiga.solver import FixedPointConfig, MonodomainProblem, fixed_point_solve

    def pulse(x, t):
        return 1.0 * (x[:, 0] < 0.1) * (t < 0.05)

    st = SpaceTimeSpace([SplineSpace.uniform(2, 64)], SplineSpace.uniform(2, 64))
    prob = MonodomainProblem(builtin_geometry("unit_interval", final_time=1.0), st, source=pulse, D=1e-3)
    t0 = time.perf_counter()
    res = fixed_point_solve(prob, FixedPointConfig(stabilization="spline_upwind", linear_solver="iterative"))
    return {"N": st.num_dof, "seconds": time.perf_counter() - t0, "sweeps": res.iterations,
            "avg_gmres": res.avg_gmres, "avg_pcg": res.avg_pcg, "converged": res.converged,
            "system": "cfg1 1D p=2 64x64, SU every sweep, iterative, source pulse 1[x<0.1] 1[t<0.05]"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-gmres", action="store_true")
    ap.add_argument("--skip-cfg4", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_ref_cpu.json"))
    args = ap.parse_args()
    import monoiga
    import numpy
    host = {"cores": os.cpu_count(), "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS", "default (all)"),
            "numpy": numpy.__version__, "reference": "monoiga %s from %s" % (monoiga.__version__, REF),
            "note": "scipy.sparse SpMM (the matvec) is single-threaded by design; numpy/OpenBLAS (P^-1) threaded"}
    out = {"host": host}
    out["fixed_point_cfg1"] = fixed_point_cfg1()
    print(json.dumps(out["fixed_point_cfg1"]), flush=True)
    for ne, ne_t in ((12, 24), (16, 32)):
        key = "apply_su_%d_%d" % (ne, ne_t)
        out[key] = time_apply(3, 3, ne, ne_t, 1e-3, True, reps=3)
        print(key, json.dumps(out[key]), flush=True)
    if not args.skip_cfg4:
        out["apply_cfg4_separable"] = time_apply(3, 3, 96, 192, 1e-3, False)
        print(json.dumps(out["apply_cfg4_separable"]), flush=True)
    if not args.skip_gmres:
        out["gmres_cfg2"] = gmres_cfg2()
        print(json.dumps(out["gmres_cfg2"]), flush=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
