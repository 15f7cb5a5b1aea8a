"""Full-size golden fixtures at the BASELINE configs, produced by the REFERENCE package here.

Run in the build container (the reference is mounted read-only) or, for cfg 4 (~65 GB of host RAM), on a
GPU box host against the identical package installed under baseline/_ref:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_fullsize.py [cfg ...]

Full-size vectors are far too large to commit, so each fixture stores size-independent summaries of
the reference's own output vectors, computed on seeded inputs the tests regenerate on the GPU box:

* ``*_idx`` / ``*_val``: the vector at a fixed sample of rows (seeded random rows, plus the first and
  last time rows' boundary points);
* ``*_rownorm``: the 2-norm of every time row (N_t values);
* ``*_rowdot``: the dot product of every time row with a seeded N(0, 1) probe vector (a checksum of
  every entry: any wrong entry anywhere moves its row's checksum).

What the reference can run at each size (SURVEY 8c limits):

* cfg 2 (2D p=3 128^2 x 256, N = 4.4 M): the full potential system at sweep 1 -- Galerkin terms,
  zero-iterate reaction and the Spline Upwind terms of the seeded front indicator (R = 6) --
  A x, P^-1 x, P^-1 A x, and ``gmres(op, f, precond=P, tol=1e-8, max_iter=300)`` with f the load vector
  of the corner-square pulse 1[x<0.1, y<0.1] 1[t<0.05] (the first fixed-point sweep's system).
* cfg 3 (3D p=2 64^3 x 128, N = 37 M, sigma = diag(1e-3, 4e-4, 4e-4)): the separable operator with the
  zero-iterate reaction (SU assembly does not fit: Kronecker collocation ~4e9 nnz), P^-1.
* cfg 4 (3D p=3 96^3 x 192, N = 188 M): the same separable operator and P^-1 (31 GB of CSR).

The Spline Upwind terms at cfgs 3/4 and the reaction mass M_R at every full size are beyond the
reference (assembly size); the tests check them on sampled rows against the pinned oracle instead.
"""

import os
import sys
import time

import numpy as np
import scipy.sparse as sp

sys.dont_write_bytecode = True
# the read-only reference checkout (build container), else the same unmodified package installed under
# baseline/_ref (a GPU box host: cfg 4 needs more RAM than the build container has)
_REF = "/root/reference/pkg/src"
if not os.path.isdir(_REF):
    _REF = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "baseline", "_ref")
sys.path.insert(0, _REF)

from monoiga.assembly import (  # noqa: E402
    KroneckerOperator, SpatialQuadratureData, UnivariateMatrices, spatial_operators, time_matrices)
from monoiga.bspline import SplineSpace, SpaceTimeSpace  # noqa: E402
from monoiga.geometry import builtin_geometry  # noqa: E402
from monoiga.linalg import FastDiagPreconditioner, build_time_pencil, generalized_eig, gmres  # noqa: E402
from monoiga.stabilization import (  # noqa: E402
    ResidualIndicator, assemble_stabilization, compute_tau, lowrank_factorize)
from monoiga.tensorops import kron_chain  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
RM = {"c1": 0.26, "a": 0.13, "c2": 0.1}
CFGS = {2: dict(d=2, p=3, ne=128, ne_t=256, sigma=(1e-3,), su=True),
        3: dict(d=3, p=2, ne=64, ne_t=128, sigma=(1e-3, 4e-4, 4e-4), su=False),
        4: dict(d=3, p=3, ne=96, ne_t=192, sigma=(1e-3,), su=False)}
NSAMPLE = 3000


def sample_rows(nt, ns, seed=3):
    """Seeded random rows + every spatial corner of the first / middle / last time rows."""
    rng = np.random.default_rng(seed)
    idx = rng.choice(nt * ns, NSAMPLE, replace=False)
    edge = np.concatenate([t * ns + np.array([0, 1, ns // 2, ns - 2, ns - 1]) for t in (0, 1, nt // 2, nt - 2, nt - 1)])
    return np.unique(np.concatenate([idx, edge]))


def summary(prefix, v, nt, ns, idx, probe):
    V = v.reshape(nt, ns)
    return {prefix + "_val": v[idx], prefix + "_rownorm": np.linalg.norm(V, axis=1),
            prefix + "_rowdot": np.einsum("ij,ij->i", V, probe.reshape(nt, ns)), prefix + "_norm": np.linalg.norm(v)}


def corner_pulse(x, t):
    """cfg-2 stimulus stand-in as a source (the reference has no u0): 1 on [0,0.1]^2 for t < 0.05."""
    return 1.0 * (x[:, 0] < 0.1) * (x[:, 1] < 0.1) * (t < 0.05)


def front(st):
    ns = st.num_space
    g1 = st.spatial[0].greville()
    gs = np.tile(g1, ns // g1.size)
    gt = st.time_greville()
    return np.clip(np.exp(-(((gs[None, :] - 0.2 - 0.5 * gt[:, None]) / 0.08) ** 2)), 0, 1)


def build(cfg):
    c = CFGS[cfg]
    d, p = c["d"], c["p"]
    st = SpaceTimeSpace([SplineSpace.uniform(p, c["ne"]) for _ in range(d)], SplineSpace.uniform(p, c["ne_t"]))
    geo = builtin_geometry({2: "unit_square", 3: "unit_cube"}[d], final_time=1.0)
    nt, ns = st.num_time, st.num_space
    W_t, M_t = time_matrices(st, 1.0)
    react = RM["a"] * RM["c1"]
    sig = np.asarray(c["sigma"])
    if sig.size == 1:
        M_s, K_s = spatial_operators(st.spatial, geo)
        terms = [(1.0, W_t, M_s), (float(sig[0]), M_t, K_s), (react, M_t, M_s)]
        sd = SpatialQuadratureData(st.spatial, geo)
        P = FastDiagPreconditioner.build(st, 1.0, 1.0, float(sig[0]), react, spatial_data=sd)
    else:   # anisotropic diagonal sigma from reference pieces
        mats = [UnivariateMatrices(s) for s in st.spatial]
        M_s = kron_chain([mats[l].mass for l in reversed(range(d))])
        K = None
        for a in range(d):
            t = sig[a] * kron_chain([mats[l].stiffness if l == a else mats[l].mass for l in reversed(range(d))])
            K = t if K is None else K + t
        terms = [(1.0, W_t, M_s), (1.0, M_t, sp.csr_matrix(K)), (react, M_t, M_s)]
        eigs = [generalized_eig(m.stiffness, m.mass) for m in mats]
        grid = np.zeros(st.spatial_shape)
        for l in range(d):
            shp = [1] * d
            shp[d - 1 - l] = eigs[l][1].size
            grid = grid + sig[l] * eigs[l][1].reshape(shp)
        P = FastDiagPreconditioner(eigs, grid.ravel(), build_time_pencil(W_t, M_t), 1.0, 1.0, react)
    rank = 0
    if c["su"]:
        th = front(st)
        ind = ResidualIndicator(th, st.time_greville(), [s.greville() for s in st.spatial], st.spatial_shape)
        lr = lowrank_factorize(ind, 0.1)
        rank = lr.rank
        terms = terms + assemble_stabilization(compute_tau(st.time), lr, st, geo, 1.0).terms()
    return st, KroneckerOperator(nt, ns, terms), P, rank


def run(cfg):
    t0 = time.perf_counter()
    st, op, P, rank = build(cfg)
    N, nt, ns = st.num_dof, st.num_time, st.num_space
    print("cfg %d: N=%d built in %.1f s (SU rank %d)" % (cfg, N, time.perf_counter() - t0, rank), flush=True)
    x = np.random.default_rng(0).uniform(-1, 1, N)
    probe = np.random.default_rng(7).standard_normal(N)
    idx = sample_rows(nt, ns)
    out = dict(cfg=cfg, N=N, nt=nt, ns=ns, su_rank=rank, idx=idx)
    t1 = time.perf_counter()
    y = op.matvec(x)
    out.update(summary("y_a", y, nt, ns, idx, probe))
    t2 = time.perf_counter()
    out.update(summary("z_pc", P.apply(x), nt, ns, idx, probe))
    t3 = time.perf_counter()
    out.update(summary("z_pca", P.apply(y), nt, ns, idx, probe))
    del y
    out["ref_seconds"] = np.array([t2 - t1, t3 - t2])
    print("cfg %d: A x %.1f s, P^-1 x %.1f s" % (cfg, t2 - t1, t3 - t2), flush=True)
    if cfg == 2:
        # the first fixed-point sweep's system: the load vector of the corner-square pulse
        from monoiga.assembly import rhs_vectors
        geo = builtin_geometry("unit_square", final_time=1.0)
        rhs, _ = rhs_vectors(st, geo, corner_pulse, np.zeros(N), 0.013)
        out.update(summary("rhs", rhs, nt, ns, idx, probe))
        t4 = time.perf_counter()
        sol, it, hist = gmres(op, rhs, precond=P, tol=1e-8, max_iter=300)
        out.update(summary("gm_x", sol, nt, ns, idx, probe))
        out.update(gm_it=it, gm_hist=np.array(hist), gm_seconds=time.perf_counter() - t4)
        print("cfg 2: gmres %d iterations in %.1f s" % (it, time.perf_counter() - t4), flush=True)
    out["reference_path"] = _REF
    tmp = os.path.join(HERE, "fullsize_cfg%d.tmp.npz" % cfg)
    np.savez_compressed(tmp, **out)
    os.replace(tmp, os.path.join(HERE, "fullsize_cfg%d.npz" % cfg))


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["3", "4", "2"]):
        run(int(c))
