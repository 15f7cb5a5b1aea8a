"""GPU: the per-rank slab operations of the space-sharded solve (CUDA backend)
match the numpy reference backend, for every rank of simulated 2-4-rank
layouts (no collectives needed: each rank's local math is checked in one
process).  Covers the z-slab operator (owned planes from an input slab with
p halo planes: global channel tables, TMA halo offset, the reaction on the
input frame) and the per-direction mode products and the y-slab time stage
of P^-1."""

import numpy as np
import pytest
import torch

from cases import RM, load
from test_sharded_cpu import NumpySlabBackend, layout_for, synthetic_case

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def input_slab(L, v):
    return np.ascontiguousarray(v.reshape(L.nt, L.n3, L.plane)[:, L.z_lo - L.h_lo:L.z_hi + L.h_hi]).ravel()


@pytest.mark.parametrize("name,world", [("case_3d_p2_front", 2), ("case_3d_p3", 2), ("synthetic", 3),
                                        ("synthetic", 4)])
@pytest.mark.parametrize("variant", ["a", "b"])
def test_slab_backend_matches_reference(name, world, variant):
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200 import sharded as sh
    g = synthetic_case() if name == "synthetic" else load(name)
    p = int(g["p"])
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, int(n)) for n in g["ne"]], mb.SplineSpace.uniform(p, int(g["ne_t"])))
    sig = np.atleast_1d(g["sigma"])
    sig = float(sig[0]) if sig.size == 1 else sig
    stab = mb.Stabilization(st, g["theta"], float(g["su_tol"]), 1.0)
    rng = np.random.default_rng(5)
    for rank in range(world):
        L = layout_for(g, rank, world)
        u = w = None
        if variant == "b":
            u, w = input_slab(L, g["u"]), input_slab(L, g["w"])
        dev = sh.DeviceSlabBackend(L, st, float(g["T"]), 1.0, sig, RM, stabilization=stab, u=u, w=w)
        ref = NumpySlabBackend(L, g, variant)
        x_in = rng.uniform(-1, 1, L.n_in)
        yd = dev.empty(L.n_own)
        dev.apply_in(torch.from_numpy(x_in).cuda(), yd)
        yr = torch.empty(L.n_own, dtype=torch.float64)
        ref.apply_in(torch.from_numpy(x_in), yr)
        assert rel(yd.cpu().numpy(), yr.numpy()) < 1e-12, (rank, variant)
        # preconditioner stages: every direction both ways on the owned / y-slab shapes, time stage
        shapes = [(0, L.nt * L.nz * L.n2, 1, L.n_own), (1, L.nt * L.nz, L.n1, L.n_own),
                  (2, L.nt, L.ny * L.n1, L.n_blk)]
        for l, outer, inner, n in shapes:
            for inv in (False, True):
                src = rng.uniform(-1, 1, n)
                od = dev.empty(n)
                dev.pc_mode(l, inv, torch.from_numpy(src).cuda(), od, outer, inner)
                orf = torch.empty(n, dtype=torch.float64)
                ref.pc_mode(l, inv, torch.from_numpy(src), orf, outer, inner)
                assert rel(od.cpu().numpy(), orf.numpy()) < 1e-12, (rank, l, inv)
        # the transposes' addressing maps (send layout for direction 2, receive layout for direction 3)
        if world > 1:
            spc_d = sh.ShardedPreconditioner(L, dev)
            spc_r = sh.ShardedPreconditioner(L, ref)
            for l, outer, inner, n_in, n_out, key in [(1, L.nt * L.nz, L.n1, L.n_own, L.n_own, "send"),
                                                      (2, L.nt, L.ny * L.n1, L.n_blk, L.n_blk, "recv")]:
                for inv in (False, True):
                    for side in ("in", "out"):
                        mp_d = getattr(spc_d, "map_" + key)
                        mp_r = getattr(spc_r, "map_" + key)
                        src = rng.uniform(-1, 1, n_in)
                        od, orf = dev.empty(n_out).zero_(), torch.zeros(n_out, dtype=torch.float64)
                        kw_d = {"imap": mp_d} if side == "in" else {"omap": mp_d}
                        kw_r = {"imap": mp_r} if side == "in" else {"omap": mp_r}
                        dev.pc_mode(l, inv, torch.from_numpy(src).cuda(), od, outer, inner, **kw_d)
                        ref.pc_mode(l, inv, torch.from_numpy(src), orf, outer, inner, **kw_r)
                        assert rel(od.cpu().numpy(), orf.numpy()) < 1e-12, (rank, l, inv, side)
        blk = rng.uniform(-1, 1, L.n_blk)
        bd = torch.from_numpy(blk).cuda()
        dev.pc_time_yslab(bd, L.y_lo, L.y_hi)
        br = torch.from_numpy(blk.copy())
        ref.pc_time_yslab(br, L.y_lo, L.y_hi)
        assert rel(bd.cpu().numpy(), br.numpy()) < 1e-12


def test_sharded_gmres_world1_nccl_equals_reference():
    """The distributed recurrence on a 1-rank NCCL group reproduces the reference GMRES."""
    import os
    import torch.distributed as dist
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200 import sharded as sh
    g = load("case_3d_p3")
    p = int(g["p"])
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, int(n)) for n in g["ne"]], mb.SplineSpace.uniform(p, int(g["ne_t"])))
    stab = mb.Stabilization(st, g["theta"], float(g["su_tol"]), 1.0)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        L = layout_for(g, 0, 1)
        be = sh.DeviceSlabBackend(L, st, float(g["T"]), 1.0, float(np.atleast_1d(g["sigma"])[0]), RM,
                                  stabilization=stab)
        sop, spc = sh.ShardedOperator(L, be), sh.ShardedPreconditioner(L, be)
        b = torch.from_numpy(g["rhs"]).cuda()
        x, it, hist = sh.sharded_gmres(sop, spc, be.vec_ops, b, tol=1e-8, max_iter=400)
        assert it == int(g["gm_a_it"])
        assert rel(x.cpu().numpy(), g["gm_a_x"]) < 1e-10
    finally:
        dist.destroy_process_group()
