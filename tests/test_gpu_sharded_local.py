"""GPU: the per-rank slab operations of the time-sharded solve (CUDA backend)
match the numpy reference backend, for every rank of simulated 2/3-rank
layouts (no collectives needed: each rank's local math is checked in one
process).  Covers time-row slicing of the operator bands, the reaction's
slab row offset, and the column-offset time stage of P^-1."""

import numpy as np
import pytest
import torch

from cases import RM, load, oracle_objects
from test_sharded_cpu import NumpySlabBackend

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name,world", [("case_2d_aniso", 2), ("case_3d_p2_front", 3), ("case_cfg1", 3)])
@pytest.mark.parametrize("variant", ["a", "b"])
def test_slab_backend_matches_reference(name, world, variant):
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200 import sharded as sh
    g = load(name)
    st_o, op_a, op_b, _, _, _ = oracle_objects(g)
    nt, ns = st_o.num_time, st_o.num_space
    p = int(g["p"])
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, int(n)) for n in g["ne"]], mb.SplineSpace.uniform(p, int(g["ne_t"])))
    sig = np.atleast_1d(g["sigma"])
    sig = float(sig[0]) if sig.size == 1 else sig
    stab = mb.Stabilization(st, g["theta"], float(g["su_tol"]), 1.0)
    rng = np.random.default_rng(5)
    for rank in range(world):
        L = sh.SlabLayout(nt, ns, p, rank, world)
        u = w = None
        if variant == "b":
            u = g["u"][L.e_lo * ns:L.e_hi * ns]
            w = g["w"][L.e_lo * ns:L.e_hi * ns]
        dev = sh.DeviceSlabBackend(L, st, float(g["T"]), 1.0, sig, RM, stabilization=stab, u=u, w=w)
        ref = NumpySlabBackend(L, g)
        if variant == "b":
            ref.op_a = op_b
        x_ext = rng.uniform(-1, 1, L.next_ * ns)
        yd = dev.empty(L.next_ * ns)
        dev.apply_ext(torch.from_numpy(x_ext).cuda(), yd)
        yr = torch.empty(L.next_ * ns, dtype=torch.float64)
        ref.apply_ext(torch.from_numpy(x_ext), yr)
        off = (L.t_lo - L.e_lo) * ns
        own = slice(off, off + L.nown * ns)
        assert rel(yd.cpu().numpy()[own], yr.numpy()[own]) < 1e-12, (rank, variant)
        # preconditioner stages
        r_own = rng.uniform(-1, 1, L.nown * ns)
        sd = dev.empty(L.nown * ns)
        dev.pc_spatial(torch.from_numpy(r_own).cuda(), sd, L.nown, inverse=False)
        sr = torch.empty(L.nown * ns, dtype=torch.float64)
        ref.pc_spatial(torch.from_numpy(r_own), sr, L.nown, inverse=False)
        assert rel(sd.cpu().numpy(), sr.numpy()) < 1e-12
        blk = rng.uniform(-1, 1, nt * L.ncols)
        bd = torch.from_numpy(blk).cuda()
        dev.pc_time(bd, L.ncols, L.s_lo)
        br = torch.from_numpy(blk.copy())
        ref.pc_time(br, L.ncols, L.s_lo)
        assert rel(bd.cpu().numpy(), br.numpy()) < 1e-12


def test_sharded_gmres_world1_nccl_equals_unsharded():
    """The distributed recurrence on a 1-rank NCCL group == the plain device GMRES."""
    import os
    import torch.distributed as dist
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200 import sharded as sh
    g = load("case_3d_p3")
    st_o = oracle_objects(g)[0]
    p = int(g["p"])
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, int(n)) for n in g["ne"]], mb.SplineSpace.uniform(p, int(g["ne_t"])))
    stab = mb.Stabilization(st, g["theta"], float(g["su_tol"]), 1.0)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        L = sh.SlabLayout(st_o.num_time, st_o.num_space, p, 0, 1)
        be = sh.DeviceSlabBackend(L, st, float(g["T"]), 1.0, float(g["sigma"][0]), RM, stabilization=stab)
        sop, spc = sh.ShardedOperator(L, be), sh.ShardedPreconditioner(L, be)
        b = torch.from_numpy(g["rhs"]).cuda()
        x, it, hist = sh.sharded_gmres(sop, spc, be.vec_ops, b, tol=1e-8, max_iter=400)
        assert it == int(g["gm_a_it"])
        assert rel(x.cpu().numpy(), g["gm_a_x"]) < 1e-10
    finally:
        dist.destroy_process_group()
