"""Generate golden fixtures by running the REFERENCE package (monoiga) here.

Run in the build container (the reference is mounted read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``monoiga`` from /root/reference/pkg/src and writes small
``.npz`` files next to this script.  Nothing on the GPU box reads the
reference; tests and the oracle only read these committed fixtures.
"""

import os
import sys

import numpy as np
import scipy.sparse as sp

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from monoiga.assembly import (  # noqa: E402
    KroneckerOperator, UnivariateMatrices, reaction_mass, spatial_operators, time_matrices)
from monoiga.bspline import SplineSpace, SpaceTimeSpace  # noqa: E402
from monoiga.geometry import builtin_geometry  # noqa: E402
from monoiga.linalg import FastDiagPreconditioner, build_time_pencil, generalized_eig, gmres  # noqa: E402
from monoiga.stabilization import (  # noqa: E402
    ResidualIndicator, assemble_stabilization, compute_tau, lowrank_factorize)
from monoiga.tensorops import kron_chain  # noqa: E402
from monoiga.solver import _Workspace, MonodomainProblem, FixedPointConfig  # noqa: E402
from monoiga.assembly import SpatialQuadratureData  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
RM = {"c1": 0.26, "a": 0.13, "c2": 0.1}


def univariate():
    out = {}
    for p in (1, 2, 3, 4):
        for ne in (1, 3, 5):
            s = SplineSpace.uniform(p, ne)
            m = UnivariateMatrices(s)
            key = "p%d_ne%d" % (p, ne)
            out[key + "_M"] = m.mass.toarray()
            out[key + "_K"] = m.stiffness.toarray()
            out[key + "_W"] = m.advection.toarray()
            out[key + "_grev"] = s.greville()
            pts = np.linspace(0, 1, 11)
            for o in range(min(p, 2) + 1):
                out[key + "_C%d" % o] = s.collocation_matrix(pts, o).toarray()
    st = SpaceTimeSpace([SplineSpace.uniform(2, 3)], SplineSpace.uniform(2, 4))
    Wt, Mt = time_matrices(st, 1.5)
    out["time_Wt"], out["time_Mt"] = Wt.toarray(), Mt.toarray()
    tau = compute_tau(SplineSpace.uniform(3, 6))
    out["tau_p3_ne6_pts"] = np.linspace(0, 1, 13)
    for k in (1, 2, 3):
        out["tau_p3_ne6_k%d" % k] = tau.evaluate(k, out["tau_p3_ne6_pts"])
    np.savez_compressed(os.path.join(HERE, "univariate.npz"), **out)


def aniso_terms(st, geo, sigma):
    """Anisotropic K_sigma from reference pieces."""
    d = st.num_spatial_dims
    mats = [UnivariateMatrices(s) for s in st.spatial]
    K = None
    for a in range(d):
        fac = [mats[l].stiffness if l == a else mats[l].mass for l in reversed(range(d))]
        t = sigma[a] * kron_chain(fac)
        K = t if K is None else K + t
    return sp.csr_matrix(K)


def case(name, d, p, ne, ne_t, T, sigma, seed, su_tol=0.3, theta=None, gm_iters=400, front=False):
    rng = np.random.default_rng(seed)
    nes = [ne] * d if np.isscalar(ne) else list(ne)
    st = SpaceTimeSpace([SplineSpace.uniform(p, n) for n in nes], SplineSpace.uniform(p, ne_t))
    geo = builtin_geometry({1: "unit_interval", 2: "unit_square", 3: "unit_cube"}[d], final_time=T)
    N, nt, ns = st.num_dof, st.num_time, st.num_space
    W_t, M_t = time_matrices(st, T)
    M_s, K_s = spatial_operators(st.spatial, geo)
    sig = np.atleast_1d(sigma)
    if sig.size == 1:
        sep = [(1.0, W_t, M_s), (float(sig[0]), M_t, K_s)]
    else:
        sep = [(1.0, W_t, M_s), (1.0, M_t, aniso_terms(st, geo, sig))]
    react = RM["a"] * RM["c1"]
    # SU terms from an indicator
    if front:
        g1 = st.spatial[0].greville()
        gs = np.tile(g1, ns // g1.size)
        gt = st.time_greville()
        th = np.clip(np.exp(-(((gs[None, :] - 0.2 - 0.5 * gt[:, None]) / 0.08) ** 2)), 0, 1)
    else:
        th = rng.random((nt, ns))
    ind = ResidualIndicator(th, st.time_greville(), [s.greville() for s in st.spatial], st.spatial_shape)
    tau = compute_tau(st.time)
    lr = lowrank_factorize(ind, su_tol)
    stab = assemble_stabilization(tau, lr, st, geo, 1.0)
    su = stab.terms()
    x = rng.uniform(-1, 1, N)
    u = rng.uniform(0, 1, N)
    w = rng.uniform(0, 0.1, N)
    rhs = rng.standard_normal(N)
    op_a = KroneckerOperator(nt, ns, sep + [(react, M_t, M_s)] + su)
    MR = reaction_mass(st, geo, RM, u, w)
    op_b = KroneckerOperator(nt, ns, sep + su, correction=MR)
    op_sep = KroneckerOperator(nt, ns, sep + [(react, M_t, M_s)])
    if sig.size == 1:
        sd = SpatialQuadratureData(st.spatial, geo)
        P = FastDiagPreconditioner.build(st, T, 1.0, float(sig[0]), react, spatial_data=sd)
    else:
        eigs = [generalized_eig(UnivariateMatrices(s).stiffness, UnivariateMatrices(s).mass) for s in st.spatial]
        grid = np.zeros(st.spatial_shape)
        for l in range(d):
            shp = [1] * d
            shp[d - 1 - l] = eigs[l][1].size
            grid = grid + sig[l] * eigs[l][1].reshape(shp)
        P = FastDiagPreconditioner(eigs, grid.ravel(), build_time_pencil(W_t, M_t), 1.0, 1.0, react)
    out = dict(d=d, p=p, ne=np.array(nes), ne_t=ne_t, T=T, sigma=sig, su_tol=su_tol, theta=th,
               x=x, u=u, w=w, rhs=rhs, su_rank=lr.rank, su_weights=lr.weights,
               y_sep=op_sep.matvec(x), y_a=op_a.matvec(x), y_b=op_b.matvec(x),
               y_mr=MR @ x, z_pc=P.apply(x), z_pc_ya=P.apply(op_a.matvec(x)))
    sol, it, hist = gmres(op_a, rhs, precond=P, tol=1e-8, max_iter=gm_iters)
    out.update(gm_a_x=sol, gm_a_it=it, gm_a_hist=np.array(hist))
    sol, it, hist = gmres(op_b, rhs, precond=P, tol=1e-8, max_iter=gm_iters)
    out.update(gm_b_x=sol, gm_b_it=it, gm_b_hist=np.array(hist))
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, "N=%d R=%d gmres a/b %d/%d" % (N, lr.rank, out["gm_a_it"], it))


if __name__ == "__main__" and len(sys.argv) == 1:
    univariate()
    case("case_2d_p2", 2, 2, (3, 2), 3, 2.0, 1e-3, seed=11)
    case("case_3d_p3", 3, 3, 3, 4, 1.0, 1e-3, seed=12)
    case("case_2d_aniso", 2, 3, (4, 3), 5, 1.0, (1e-3, 4e-4), seed=13)
    case("case_1d_p1", 1, 1, 6, 5, 1.0, 1e-2, seed=14)
    case("case_cfg1", 1, 2, 64, 64, 1.0, 1e-3, seed=0, su_tol=0.1, front=True)
    case("case_3d_p2_front", 3, 2, (6, 4, 3), 8, 1.0, (1e-3, 4e-4, 4e-4), seed=15, su_tol=0.1, front=True)


def pulse_source(x, t):
    """Stimulus stand-in (the reference cannot take u0 != 0)."""
    return 1.0 * (x[:, 0] < 0.1) * (t < 0.05)


def fixed_point_cases():
    from monoiga.solver import fixed_point_solve
    from monoiga.stabilization import compute_theta
    out = {}
    cases = [("fp_1d_off", 1, 2, 12, 12, "off"), ("fp_1d_su", 1, 2, 12, 12, "spline_upwind"),
             ("fp_2d_su", 2, 2, (6, 5), 8, "spline_upwind")]
    for name, d, p, ne, ne_t, stab in cases:
        nes = [ne] * d if np.isscalar(ne) else list(ne)
        st = SpaceTimeSpace([SplineSpace.uniform(p, n) for n in nes], SplineSpace.uniform(p, ne_t))
        geo = builtin_geometry({1: "unit_interval", 2: "unit_square"}[d], final_time=1.0)
        prob = MonodomainProblem(geo, st, source=pulse_source, D=1e-3)
        cfg = FixedPointConfig(stabilization=stab, linear_solver="iterative")
        res = fixed_point_solve(prob, cfg)
        from monoiga.assembly import rhs_vectors
        fv, _ = rhs_vectors(st, geo, pulse_source, np.zeros(st.num_dof), prob.b)
        out[name + "_f"] = fv
        out.update({name + "_u": res.u, name + "_w": res.w, name + "_it": res.iterations,
                    name + "_inc": np.array(res.increments), name + "_gm": np.array(res.gmres_iterations),
                    name + "_pcg": np.array(res.pcg_iterations), name + "_d": d, name + "_p": p,
                    name + "_ne": np.array(nes), name + "_ne_t": ne_t})
        print(name, "sweeps", res.iterations, "gmres", res.gmres_iterations[:5])
    # compute_theta at a random state (2D)
    rng = np.random.default_rng(21)
    st = SpaceTimeSpace([SplineSpace.uniform(2, 5), SplineSpace.uniform(3, 4)], SplineSpace.uniform(2, 6))
    geo = builtin_geometry("unit_square", final_time=2.0)
    prob = MonodomainProblem(geo, st, source=pulse_source, D=1e-2)
    u = rng.uniform(0, 1, st.num_dof)
    w = rng.uniform(0, 0.1, st.num_dof)
    th = compute_theta(prob, u, w)
    out.update(theta_u=u, theta_w=w, theta_values=th.values)
    np.savez_compressed(os.path.join(HERE, "fixed_point.npz"), **out)


def theta_cases():
    """compute_theta at random states on equal-degree spaces (the device path's domain)."""
    from monoiga.geometry import box_geometry
    from monoiga.stabilization import compute_theta
    out = {}
    rng = np.random.default_rng(33)
    cases = [("th3d", 2, (4, 3, 5), 6, (1.0, 0.5, 2.0), 2.0, True, 1e-2),
             ("th1d", 3, (9,), 7, (1.5,), 1.0, False, 1e-3)]
    for name, p, nes, ne_t, L, T, with_src, D in cases:
        st = SpaceTimeSpace([SplineSpace.uniform(p, n) for n in nes], SplineSpace.uniform(p, ne_t))
        geo = box_geometry(list(L), final_time=T)
        prob = MonodomainProblem(geo, st, source=pulse_source if with_src else None, D=D)
        u = rng.uniform(0, 1, st.num_dof)
        w = rng.uniform(0, 0.1, st.num_dof)
        th = compute_theta(prob, u, w)
        out.update({name + "_u": u, name + "_w": w, name + "_values": th.values, name + "_p": p,
                    name + "_ne": np.array(nes), name + "_ne_t": ne_t, name + "_L": np.array(L), name + "_T": T,
                    name + "_src": int(with_src), name + "_D": D})
        print(name, th.values.shape, float(th.values.max()))
    np.savez_compressed(os.path.join(HERE, "theta.npz"), **out)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "fixed_point":
    fixed_point_cases()


def fixed_point_3d_cases():
    """3D box fixed-point solves with Spline Upwind (p = 2 and 3, ~2-3k DoFs, GMRES iterative):
    the 3D counterparts of fixed_point_cases, compared sweep for sweep on the device."""
    from monoiga.solver import fixed_point_solve
    from monoiga.assembly import rhs_vectors
    out = {}
    cases = [("fp_3d_p2_su", 3, 2, (6, 5, 4), 8, "spline_upwind", 1e-2),
             ("fp_3d_p3_su", 3, 3, (4, 3, 3), 6, "spline_upwind", 1e-2),
             ("fp_3d_p2_off", 3, 2, (6, 5, 4), 8, "off", 1e-2)]
    for name, d, p, nes, ne_t, stab, D in cases:
        st = SpaceTimeSpace([SplineSpace.uniform(p, n) for n in nes], SplineSpace.uniform(p, ne_t))
        geo = builtin_geometry("unit_cube", final_time=1.0)
        prob = MonodomainProblem(geo, st, source=pulse_source, D=D)
        res = fixed_point_solve(prob, FixedPointConfig(stabilization=stab, linear_solver="iterative"))
        fv, _ = rhs_vectors(st, geo, pulse_source, np.zeros(st.num_dof), prob.b)
        out.update({name + "_u": res.u, name + "_w": res.w, name + "_it": res.iterations,
                    name + "_inc": np.array(res.increments), name + "_gm": np.array(res.gmres_iterations),
                    name + "_pcg": np.array(res.pcg_iterations), name + "_d": d, name + "_p": p,
                    name + "_ne": np.array(nes), name + "_ne_t": ne_t, name + "_D": D, name + "_f": fv})
        print(name, "N", st.num_dof, "sweeps", res.iterations, "gmres", res.gmres_iterations[:5], flush=True)
    np.savez_compressed(os.path.join(HERE, "fixed_point_3d.npz"), **out)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "fixed_point_3d":
    fixed_point_3d_cases()

if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "theta":
    theta_cases()


def warped_cube_geometry(final_time=1.0):
    """A curved 3D map: degree-2 tensor spline whose control net is the Greville grid of the unit
    cube pushed through a smooth bijection (det J > 0)."""
    from monoiga.geometry import GeometryMap
    spaces = [SplineSpace.uniform(2, 2) for _ in range(3)]
    g = [s.greville() for s in spaces]
    Z, Y, X = np.meshgrid(g[2], g[1], g[0], indexing="ij")
    x = X + 0.08 * np.sin(np.pi * Y) * (1.0 + Z)
    y = Y * (1.0 + 0.25 * X) + 0.05 * Z
    z = Z * (1.0 + 0.2 * X * Y) - 0.06 * np.sin(np.pi * X)
    ctrl = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)
    return GeometryMap(spaces, ctrl, final_time=final_time)


def smooth_source(x, t):
    return np.exp(-((x[:, 0] - 0.3) ** 2 + (x[:, 1] - 0.2) ** 2) / 0.05) * (t < 0.4)


def mapped_cases():
    """Mapped (non-affine) geometries: SpatialQuadratureData mass/stiffness, the reaction mass, the
    separable-weight preconditioner, GMRES and the load vector."""
    from monoiga.assembly import rhs_vectors
    from monoiga.geometry import builtin_geometry, save_geometry
    out = {}
    geos = {"annulus": builtin_geometry("ellipse_annulus", final_time=1.0), "warped": warped_cube_geometry()}
    for key, geo in geos.items():
        save_geometry(geo, os.path.join(HERE, "geo_%s.txt" % key))
    cases = [("m2d", "annulus", 2, (8, 3), 4, 1e-3, 41), ("m3d_p2", "warped", 2, (3, 3, 4), 3, 1e-2, 42),
             ("m3d_p3", "warped", 3, (2, 2, 3), 3, 1e-2, 43)]
    for name, gkey, p, nes, ne_t, D, seed in cases:
        rng = np.random.default_rng(seed)
        geo = geos[gkey]
        T = 1.0
        st = SpaceTimeSpace([SplineSpace.uniform(p, n) for n in nes], SplineSpace.uniform(p, ne_t))
        N, nt, ns = st.num_dof, st.num_time, st.num_space
        sd = SpatialQuadratureData(st.spatial, geo)
        M_s, K_s = sd.mass(), sd.stiffness()
        W_t, M_t = time_matrices(st, T)
        react = RM["a"] * RM["c1"]
        x = rng.uniform(-1, 1, N)
        u = rng.uniform(0, 1, N)
        w = rng.uniform(0, 0.1, N)
        rhs = rng.standard_normal(N)
        op_a = KroneckerOperator(nt, ns, [(1.0, W_t, M_s), (D, M_t, K_s), (react, M_t, M_s)])
        MR = reaction_mass(st, geo, RM, u, w, spatial_data=sd)
        op_b = KroneckerOperator(nt, ns, [(1.0, W_t, M_s), (D, M_t, K_s)], correction=MR)
        P = FastDiagPreconditioner.build(st, T, 1.0, D, react, spatial_data=sd)
        wm, wk = FastDiagPreconditioner._separable_weights(sd)
        f, _ = rhs_vectors(st, geo, smooth_source, np.zeros(N), 0.013, spatial_data=sd)
        rec = {"geo": gkey, "p": p, "ne": np.array(nes), "ne_t": ne_t, "D": D, "x": x, "u": u, "w": w,
               "rhs": rhs, "M_s": M_s.toarray(), "K_s": K_s.toarray(), "y_a": op_a.matvec(x), "y_b": op_b.matvec(x),
               "y_mr": MR @ x, "z_pc": P.apply(x), "f": f, "detj": sd.detj, "xq": sd.xgrid}
        for l in range(len(nes)):
            rec["wmass%d" % l], rec["wstiff%d" % l] = wm[l], wk[l]
        sol, it, hist = gmres(op_a, rhs, precond=P, tol=1e-8, max_iter=400)
        rec.update(gm_a_x=sol, gm_a_it=it, gm_a_hist=np.array(hist))
        sol, it, hist = gmres(op_b, rhs, precond=P, tol=1e-8, max_iter=400)
        rec.update(gm_b_x=sol, gm_b_it=it, gm_b_hist=np.array(hist))
        out.update({name + "_" + k: v for k, v in rec.items()})
        print(name, "N=%d gmres a/b %d/%d" % (N, rec["gm_a_it"], it), "detJ in [%.3f, %.3f]" % (sd.detj.min(), sd.detj.max()))
    # full fixed-point solve on the annulus (Galerkin: the residual indicator needs map Hessians)
    from monoiga.solver import fixed_point_solve
    st = SpaceTimeSpace([SplineSpace.uniform(2, 8), SplineSpace.uniform(2, 3)], SplineSpace.uniform(2, 8))
    prob = MonodomainProblem(geos["annulus"], st, source=smooth_source, D=1e-3)
    res = fixed_point_solve(prob, FixedPointConfig(stabilization="off", linear_solver="iterative"))
    out.update(fp_u=res.u, fp_w=res.w, fp_it=res.iterations, fp_gm=np.array(res.gmres_iterations),
               fp_pcg=np.array(res.pcg_iterations), fp_inc=np.array(res.increments))
    print("fp annulus sweeps", res.iterations, "gmres", res.gmres_iterations, "pcg", res.pcg_iterations[:6])
    np.savez_compressed(os.path.join(HERE, "mapped.npz"), **out)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "mapped":
    mapped_cases()


def mapped_su_cases():
    """Spline Upwind on mapped geometries (the reference's own SU-vs-Galerkin setting, acceptance
    criterion 7, is the ellipse annulus): the residual indicator with the mapped Laplacian (map
    Hessians), the SU Kronecker terms (SpatialQuadratureData on cells split at the spatial Greville
    abscissae, p+2 points, |det J|-weighted), the operator with them, and a full SU fixed-point
    solve."""
    from monoiga.solver import fixed_point_solve
    from monoiga.stabilization import compute_theta
    out = {}
    geos = {"annulus": builtin_geometry("ellipse_annulus", final_time=1.0), "warped": warped_cube_geometry()}
    cases = [("s2d", "annulus", 2, (8, 3), 4, 1e-3, 51), ("s2d_p3", "annulus", 3, (6, 4), 5, 1e-3, 52),
             ("s3d_p2", "warped", 2, (3, 3, 4), 3, 1e-2, 53), ("s3d_p3", "warped", 3, (2, 2, 3), 3, 1e-2, 54)]
    for name, gkey, p, nes, ne_t, D, seed in cases:
        rng = np.random.default_rng(seed)
        geo = geos[gkey]
        st = SpaceTimeSpace([SplineSpace.uniform(p, n) for n in nes], SplineSpace.uniform(p, ne_t))
        N, nt, ns = st.num_dof, st.num_time, st.num_space
        u = rng.uniform(0, 1, N)
        w = rng.uniform(0, 0.1, N)
        x = rng.uniform(-1, 1, N)
        prob = MonodomainProblem(geo, st, source=smooth_source, D=D)
        ind = compute_theta(prob, u, w)
        tau = compute_tau(st.time)
        # the operator from a random indicator (rank > 1 at tol 0.3)
        thr = rng.random((nt, ns))
        ind_r = ResidualIndicator(thr, st.time_greville(), [s.greville() for s in st.spatial], st.spatial_shape)
        lr = lowrank_factorize(ind_r, 0.3)
        stab = assemble_stabilization(tau, lr, st, geo, 1.0)
        sd = SpatialQuadratureData(st.spatial, geo)
        M_s, K_s = sd.mass(), sd.stiffness()
        W_t, M_t = time_matrices(st, 1.0)
        react = RM["a"] * RM["c1"]
        op = KroneckerOperator(nt, ns, [(1.0, W_t, M_s), (D, M_t, K_s), (react, M_t, M_s)] + stab.terms())
        rec = {"geo": gkey, "p": p, "ne": np.array(nes), "ne_t": ne_t, "D": D, "u": u, "w": w, "x": x,
               "theta": ind.values, "theta_r": thr, "su_rank": lr.rank, "y": op.matvec(x)}
        for r in range(lr.rank):
            rec["ss%d" % r] = stab.space_mats[r].toarray()
        out.update({name + "_" + k: v for k, v in rec.items()})
        print(name, "N=%d R=%d theta max %.3f" % (N, lr.rank, ind.values.max()))
    st = SpaceTimeSpace([SplineSpace.uniform(2, 8), SplineSpace.uniform(2, 3)], SplineSpace.uniform(2, 8))
    prob = MonodomainProblem(geos["annulus"], st, source=smooth_source, D=1e-3)
    res = fixed_point_solve(prob, FixedPointConfig(stabilization="spline_upwind", linear_solver="iterative"))
    out.update(fp_u=res.u, fp_w=res.w, fp_it=res.iterations, fp_gm=np.array(res.gmres_iterations),
               fp_pcg=np.array(res.pcg_iterations), fp_inc=np.array(res.increments))
    print("fp SU annulus sweeps", res.iterations, "gmres", res.gmres_iterations, "pcg", res.pcg_iterations[:6])
    np.savez_compressed(os.path.join(HERE, "mapped_su.npz"), **out)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "mapped_su":
    mapped_su_cases()
