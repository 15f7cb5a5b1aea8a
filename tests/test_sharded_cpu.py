"""Space-sharded orchestration (z-plane halo exchange, all-to-all transposes to
y-slabs, allreduce'd GMRES) on CPU with the gloo backend, world_size 2-8.

The product orchestration (paper_2311_17500_b200/sharded.py) runs unchanged;
the local slab operations are supplied by a numpy reference backend built on
the reference-pinned oracle, so these tests check the data movement and the
distributed recurrence, not the CUDA kernels (those are covered by the GPU
tests in test_gpu_sharded_local.py).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from cases import RM, load, oracle_objects
from oracle import problem as oprob
from oracle.krylov import gmres as ogmres
from oracle.splines import make_space_time


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def synthetic_case(ne=(3, 3, 10), ne_t=4, p=2, sigma=(1e-2, 4e-3, 4e-3)):
    """A 3D case with enough z planes for 3-4 ranks; expected values from the oracle."""
    st = make_space_time(3, p, list(ne), ne_t)
    rng = np.random.default_rng(11)
    theta = oprob.front_indicator(st)
    g = {"d": np.array(3), "p": np.array(p), "ne": np.array(ne), "ne_t": np.array(ne_t), "T": np.array(1.0),
         "sigma": np.array(sigma), "su_tol": np.array(0.1), "theta": theta,
         "u": rng.uniform(0, 1, st.num_dof), "w": rng.uniform(0, 0.1, st.num_dof),
         "x": rng.uniform(-1, 1, st.num_dof), "rhs": rng.uniform(-1, 1, st.num_dof)}
    _, op_a, _, P, _, _ = oracle_objects(g)
    g["y_a"] = op_a.matvec(g["x"])
    g["z_pc"] = P.apply(g["x"])
    xs, it, _ = ogmres(op_a, g["rhs"], precond=P, tol=1e-8, max_iter=400)
    g["gm_a_x"], g["gm_a_it"] = xs, np.array(it)
    return g


class NumpySlabBackend:
    """Reference local operations for one rank (test infrastructure)."""

    def __init__(self, layout, g, variant="a"):
        from paper_2311_17500_b200 import factors
        from paper_2311_17500_b200.spaces import SpaceTimeSpace, SplineSpace
        self.L = layout
        _, op_a, op_b, _, _, _ = oracle_objects(g)
        self.op = op_b if variant == "b" else op_a
        p = int(g["p"])
        st = SpaceTimeSpace([SplineSpace.uniform(p, int(n)) for n in g["ne"]],
                            SplineSpace.uniform(p, int(g["ne_t"])))
        self.st = st
        self.eigs = factors.spatial_eigs(st)
        self.pen = factors.time_pencil(st, float(g["T"]))
        d = len(st.spatial)
        sig = np.atleast_1d(g["sigma"])
        sig = np.repeat(sig, d) if sig.size == 1 else sig
        mu = np.zeros(st.spatial_shape)
        for l in range(d):
            shp = [1] * d
            shp[d - 1 - l] = -1
            mu = mu + sig[l] * self.eigs[l][1].reshape(shp)
        self.mu = mu + RM["a"] * RM["c1"]               # (n3, n2, n1)
        self.vec_ops = TorchVecOps()

    def empty(self, n):
        return torch.empty(n, dtype=torch.float64)

    def apply_in(self, x_in, y_own):
        L = self.L
        xg = np.zeros((L.nt, L.n3, L.plane))
        xg[:, L.z_lo - L.h_lo:L.z_hi + L.h_hi] = x_in.numpy().reshape(L.nt, L.nz_in, L.plane)
        yg = self.op.matvec(xg.ravel()).reshape(L.nt, L.n3, L.plane)
        y_own.copy_(torch.from_numpy(np.ascontiguousarray(yg[:, L.z_lo:L.z_hi]).ravel()))

    def index_map(self, m):
        return m

    def pc_mode(self, l, inverse, src, dst, outer, inner, imap=None, omap=None):
        """mi_pc_mode / mi_pc_mode_mapped: element (o, r, c) at map[r, 0] + o map[r, 1] + c."""
        U = self.eigs[l][0]
        n = U.shape[0]
        A = U if inverse else U.T
        o = np.arange(outer)[:, None, None]
        r = np.arange(n)[None, :, None]
        c = np.arange(inner)[None, None, :]

        def addr(m):
            return (o * n + r) * inner + c if m is None else m[:, 0][r] + o * m[:, 1][r] + c

        X = src.numpy()[addr(imap)]
        Y = np.einsum("ij,ojc->oic", A, X)
        out = dst.numpy()
        out[addr(omap)] = Y

    def pc_time_yslab(self, blk, y_lo, y_hi):
        pen, L = self.pen, self.L
        mu = np.ascontiguousarray(self.mu[:, y_lo:y_hi, :]).ravel()
        ncols = mu.size
        Y = pen.Q.T @ blk.numpy().reshape(L.nt, ncols)
        diag, off, part = pen.coupling()
        a = diag[:, None] + mu[None]
        e = diag[part][:, None] + mu[None]
        b = off[:, None]
        c = off[part][:, None]
        det = a * e - b * c

        def Dinv(v):
            return (e * v - b * v[part]) / det

        gb = pen.g[:, None] * np.ones_like(mu)[None]
        dy, db = Dinv(Y[:-1]), Dinv(gb)
        xl = (Y[-1] - np.sum(pen.g_low[:, None] * dy, 0)) / (pen.sigma + mu - np.sum(pen.g_low[:, None] * db, 0))
        Z = pen.Q @ np.vstack([dy - db * xl[None], xl[None]])
        blk.copy_(torch.from_numpy(np.ascontiguousarray(Z).ravel()))


class TorchVecOps:
    def dots(self, V, k, w, out):
        out[:k] = V[:k] @ w

    def sub_comb(self, V, k, h, w):
        w -= h[:k] @ V[:k]

    def normalize(self, src, nrm2, dst):
        dst.copy_(src / torch.sqrt(nrm2[0]))

    def comb(self, V, k, y, x0, out):
        out.copy_((x0 if x0 is not None else 0.0) + y[:k] @ V[:k])


def layout_for(g, rank, world):
    from paper_2311_17500_b200 import sharded as sh
    p = int(g["p"])
    n = [int(v) + p for v in g["ne"]]
    nt = int(g["ne_t"]) + p - 1
    return sh.ZSlabLayout(nt, n, p, rank, world)


def _worker(rank, world, port, q, g):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_17500_b200 import sharded as sh
        L = layout_for(g, rank, world)
        be = NumpySlabBackend(L, g)
        sop = sh.ShardedOperator(L, be)
        spc = sh.ShardedPreconditioner(L, be)
        x = torch.from_numpy(np.ascontiguousarray(L.own_slice(g["x"])))
        y = torch.empty_like(x)
        z = torch.empty_like(x)
        sop.apply_device(x, y)
        spc.apply_device(x, z)
        b = torch.from_numpy(np.ascontiguousarray(L.own_slice(g["rhs"])))
        xs, it, hist = sh.sharded_gmres(sop, spc, be.vec_ops, b, tol=1e-8, max_iter=400)
        q.put((rank, y.numpy(), z.numpy(), xs.numpy(), it, hist))
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, "error", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _gather(g, res, key_index, world):
    """Reassemble owned z-slabs of every rank into a global (N_t, n_3, n_2, n_1) vector."""
    L0 = layout_for(g, 0, world)
    out = np.zeros((L0.nt, L0.n3, L0.plane))
    for r in res:
        L = layout_for(g, r[0], world)
        out[:, L.z_lo:L.z_hi] = r[key_index].reshape(L.nt, L.nz, L.plane)
    return out.ravel()


# "synthetic8": the BASELINE's largest rank count (8 z slabs of 2 planes, 8 y-column ranges of 1)
CASES = [(2, "case_3d_p2_front"), (2, "case_3d_p3"), (3, "synthetic"), (4, "synthetic"), (8, "synthetic8")]


@pytest.mark.parametrize("world,CASE", CASES)
def test_space_sharded_apply_and_gmres_gloo(world, CASE):
    if CASE == "synthetic8":
        g = synthetic_case(ne=(3, 6, 14))
    else:
        g = synthetic_case() if CASE == "synthetic" else load(CASE)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, g)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for r in res:
        assert not (isinstance(r[1], str) and r[1] == "error"), r[2]
    res.sort(key=lambda r: r[0])
    # halo exchange: sharded A x == global A x
    y = _gather(g, res, 1, world)
    assert np.linalg.norm(y - g["y_a"]) / np.linalg.norm(g["y_a"]) < 1e-13
    # all-to-all transposes: sharded P^-1 x == reference P^-1 x
    z = _gather(g, res, 2, world)
    assert np.linalg.norm(z - g["z_pc"]) / np.linalg.norm(g["z_pc"]) < 1e-12
    # allreduce'd GMRES: identical iteration count on every rank, solution matches the reference
    assert {r[4] for r in res} == {int(g["gm_a_it"])}
    xs = _gather(g, res, 3, world)
    assert np.linalg.norm(xs - g["gm_a_x"]) / np.linalg.norm(g["gm_a_x"]) < 1e-10


def test_layout_rejects_too_many_ranks():
    from paper_2311_17500_b200 import sharded as sh
    with pytest.raises(ValueError):
        sh.ZSlabLayout(5, [6, 6, 5], 3, 0, 2)      # 5 planes cannot give 2 ranks a 3-plane halo
    L = sh.ZSlabLayout(5, [6, 6, 9], 3, 1, 3)
    assert (L.z_lo, L.z_hi, L.h_lo, L.h_hi, L.nz_in) == (3, 6, 3, 3, 9)
    assert (L.y_lo, L.y_hi) == (2, 4)
