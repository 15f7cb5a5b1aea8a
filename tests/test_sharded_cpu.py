"""Time-sharded orchestration (halo exchange, all-to-all transposes, allreduce'd
GMRES) on CPU with the gloo backend, world_size 2 and 3.

The product orchestration (paper_2311_17500_b200/sharded.py) runs unchanged;
the local slab operations are supplied by a numpy reference backend built on
the reference-pinned oracle, so these tests check the data movement and the
distributed recurrence, not the CUDA kernels (those are covered by the GPU
parity tests).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from cases import RM, load, oracle_objects



def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class NumpySlabBackend:
    """Reference local operations for one rank (test infrastructure)."""

    def __init__(self, layout, g):
        from paper_2311_17500_b200 import factors
        from paper_2311_17500_b200.spaces import SpaceTimeSpace, SplineSpace
        self.L = layout
        st_o, self.op_a, _, _, _, _ = oracle_objects(g)
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
        self.mu = mu.ravel() + RM["a"] * RM["c1"]
        self.vec_ops = TorchVecOps()

    def empty(self, n):
        return torch.empty(n, dtype=torch.float64)

    def apply_ext(self, x_ext, y_ext):
        L = self.L
        xg = np.zeros(L.nt * L.ns)
        xg[L.e_lo * L.ns:L.e_hi * L.ns] = x_ext.numpy()
        y_ext.copy_(torch.from_numpy(self.op_a.matvec(xg)[L.e_lo * L.ns:L.e_hi * L.ns]))

    def _mode(self, A, X, ax):
        t = np.moveaxis(X, ax, 0)
        o = (A @ t.reshape(t.shape[0], -1)).reshape((A.shape[0],) + t.shape[1:])
        return np.moveaxis(o, 0, ax)

    def pc_spatial(self, src, dst, nrows, inverse):
        d = len(self.st.spatial)
        X = src.numpy().reshape((nrows,) + self.st.spatial_shape)
        for l in range(d):
            U = self.eigs[l][0]
            X = self._mode(U if inverse else U.T, X, 1 + (d - 1 - l))
        dst.copy_(torch.from_numpy(np.ascontiguousarray(X).ravel()))

    def pc_time(self, blk, ncols, col0):
        pen = self.pen
        Y = pen.Q.T @ blk.numpy().reshape(self.L.nt, ncols)
        mu = self.mu[col0:col0 + ncols]
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


def _worker(rank, world, port, q, CASE):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_17500_b200 import sharded as sh
        g = load(CASE)
        st_o, op_a, _, P, _, _ = oracle_objects(g)
        nt, ns = st_o.num_time, st_o.num_space
        L = sh.SlabLayout(nt, ns, int(g["p"]), rank, world)
        be = NumpySlabBackend(L, g)
        sop = sh.ShardedOperator(L, be)
        spc = sh.ShardedPreconditioner(L, be)
        x = torch.from_numpy(g["x"][L.t_lo * ns:L.t_hi * ns].copy())
        y = torch.empty_like(x)
        z = torch.empty_like(x)
        sop.apply_device(x, y)
        spc.apply_device(x, z)
        b = torch.from_numpy(g["rhs"][L.t_lo * ns:L.t_hi * ns].copy())
        xs, it, hist = sh.sharded_gmres(sop, spc, be.vec_ops, b, tol=1e-8, max_iter=400)
        q.put((rank, L.t_lo, L.t_hi, y.numpy(), z.numpy(), xs.numpy(), it, hist))
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        q.put((rank, "error", repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,CASE", [(2, "case_2d_aniso"), (3, "case_3d_p2_front"), (4, "case_cfg1")])
def test_time_sharded_apply_and_gmres_gloo(world, CASE):
    g = load(CASE)
    st, op_a, _, P, _, _ = oracle_objects(g)
    ns = st.num_space
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, CASE)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for r in res:
        assert r[1] != "error", r
    res.sort(key=lambda r: r[0])
    y = np.concatenate([r[3] for r in res])
    z = np.concatenate([r[4] for r in res])
    xs = np.concatenate([r[5] for r in res])
    # halo exchange: sharded A x == global A x
    yref = g["y_a"]
    assert np.linalg.norm(y - yref) / np.linalg.norm(yref) < 1e-13
    # all-to-all transposes: sharded P^-1 x == reference P^-1 x
    zref = g["z_pc"]
    assert np.linalg.norm(z - zref) / np.linalg.norm(zref) < 1e-12
    # allreduce'd GMRES: identical iteration count on every rank, solution matches the reference
    its = {r[6] for r in res}
    assert its == {int(g["gm_a_it"])}
    assert np.linalg.norm(xs - g["gm_a_x"]) / np.linalg.norm(g["gm_a_x"]) < 1e-10
    assert [r[1] for r in res] == sorted(r[1] for r in res)
