"""Space-sharded solve over torch.distributed: one process per GPU.

Each rank owns a contiguous slab of planes [z_lo, z_hi) of the slowest spatial
direction (direction 3) for ALL time rows: a vector slab is the C-order
(N_t, z_hi - z_lo, n_2, n_1) block.  Sharding space instead of time keeps every
rank's operator sweep over the full time axis, where the tensor-core stencil
amortises its per-block start-up (a time slab of N_t/G rows would spend most
of each block on start-up and halo rows).  The exchanges are exactly the ones
the path needs:

* operator A: a p-plane halo of x from each z neighbour (send/recv, all time
  rows), then the local z-slab operator (stencil, time filter, reaction on
  the input slab) writes the owned planes directly.  (u, w halos are exchanged
  once when the operator is built.)
* preconditioner P^-1: the direction-1 and -2 eigenvector transforms on the
  owned slab, an all-to-all transpose to y-slabs (every rank then holds all
  z planes and all time rows of n_2/G y-columns), the direction-3 transform
  and the time stage (Q^T, arrowhead, Q) locally, the inverse direction-3
  transform, the inverse all-to-all, the inverse direction-2/1 transforms.
  The direction-2/3 transforms write / read the all-to-all buffers in their
  send / receive layouts (addressing maps), so nothing packs or unpacks.
* GMRES: the CGS2 dot products and norms are summed with all_reduce; the
  Hessenberg recurrence is replicated on every rank (krylov.gmres_core).

The orchestration is backend-agnostic: ``DeviceSlabBackend`` runs the CUDA
kernels of libmonoiga_b200 (NCCL on the GPU box); the CPU tests plug in a
reference backend with the gloo process group (tests/test_sharded_cpu.py).
"""

import torch
import torch.distributed as dist

from .krylov import DeviceVecOps, gmres_core


def split(n, parts):
    """Contiguous balanced partition of range(n) into ``parts`` slabs."""
    base, extra = divmod(n, parts)
    bounds = [0]
    for r in range(parts):
        bounds.append(bounds[-1] + base + (1 if r < extra else 0))
    return bounds


class ZSlabLayout:
    """Ownership of one rank: z planes [z_lo, z_hi) (vectors, A) and y columns [y_lo, y_hi)
    (the transposed layout inside P^-1).  ``n = (n_1, n_2, n_3)``, ``halo`` = spatial degree p."""

    def __init__(self, nt, n, halo, rank, world):
        n1, n2, n3 = (int(v) for v in n)
        if n3 < world * max(halo, 1):
            raise ValueError("too few z planes (%d) for %d ranks with halo %d" % (n3, world, halo))
        if n2 < world:
            raise ValueError("too few y columns (%d) for %d ranks" % (n2, world))
        self.nt, self.n1, self.n2, self.n3 = int(nt), n1, n2, n3
        self.halo, self.rank, self.world = int(halo), rank, world
        self.zs = split(n3, world)
        self.ys = split(n2, world)
        self.z_lo, self.z_hi = self.zs[rank], self.zs[rank + 1]
        self.y_lo, self.y_hi = self.ys[rank], self.ys[rank + 1]
        self.h_lo = min(self.halo, self.z_lo)
        self.h_hi = min(self.halo, n3 - self.z_hi)

    @property
    def nz(self):
        return self.z_hi - self.z_lo

    @property
    def nz_in(self):
        return self.nz + self.h_lo + self.h_hi

    @property
    def ny(self):
        return self.y_hi - self.y_lo

    @property
    def plane(self):
        return self.n1 * self.n2

    @property
    def n_own(self):
        return self.nt * self.nz * self.plane

    @property
    def n_in(self):
        return self.nt * self.nz_in * self.plane

    @property
    def n_blk(self):
        return self.nt * self.n3 * self.ny * self.n1

    def own_slice(self, x_global):
        """This rank's slab of a global (N_t, n_3, n_2, n_1) vector (any array type)."""
        return x_global.reshape(self.nt, self.n3, self.plane)[:, self.z_lo:self.z_hi].reshape(-1)


def _staged(t, group=None):
    """CUDA tensors under a gloo group are exchanged through host copies (functional runs of several
    ranks on one GPU; NCCL moves device memory directly)."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def _all_to_all(out, inp, out_splits, in_splits, group=None):
    if _staged(inp, group):
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=group)
        out.copy_(o)
    else:
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)


def exchange_halo(L, x_own, x_in, group=None):
    """x_in = [h_lo planes from the left | owned planes | h_hi planes from the right], all time rows."""
    nt, P = L.nt, L.plane
    xo = x_own.view(nt, L.nz, P)
    xi = x_in.view(nt, L.nz_in, P)
    xi[:, L.h_lo:L.h_lo + L.nz].copy_(xo)
    if L.world == 1:
        return x_in
    ops, recv = [], []
    h = L.halo
    dev = "cpu" if _staged(x_own, group) else x_own.device
    if L.rank > 0:
        snd = xo[:, :h].contiguous().to(dev)           # my first planes = the left neighbour's upper halo
        rcv = torch.empty(nt, L.h_lo, P, dtype=x_own.dtype, device=dev)
        ops += [dist.P2POp(dist.isend, snd, L.rank - 1, group), dist.P2POp(dist.irecv, rcv, L.rank - 1, group)]
        recv.append((rcv, 0))
    if L.rank < L.world - 1:
        snd_r = xo[:, L.nz - h:].contiguous().to(dev)
        rcv_r = torch.empty(nt, L.h_hi, P, dtype=x_own.dtype, device=dev)
        ops += [dist.P2POp(dist.isend, snd_r, L.rank + 1, group), dist.P2POp(dist.irecv, rcv_r, L.rank + 1, group)]
        recv.append((rcv_r, L.h_lo + L.nz))
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    for buf, at in recv:
        xi[:, at:at + buf.shape[1]].copy_(buf)
    return x_in


class ShardedOperator:
    """y_own = (A x)_own: p-plane halo exchange + the local z-slab operator (``apply_device``)."""

    def __init__(self, layout, backend, group=None):
        self.layout, self.backend, self.group = layout, backend, group
        self.x_in = backend.empty(layout.n_in)

    def apply_device(self, x_own, y_own):
        if self.layout.world == 1:                   # no halo: the owned slab is the input slab
            self.backend.apply_in(x_own, y_own)
            return
        exchange_halo(self.layout, x_own, self.x_in, self.group)
        self.backend.apply_in(self.x_in, y_own)


class ShardedPreconditioner:
    """z_own = (P^-1 r)_own with two all-to-all transposes (``apply_device``).

    The direction-2 and -3 mode products read and write the all-to-all send / receive layouts
    directly through addressing maps (mi_pc_mode_mapped): element (o, r, c) of a mode product lives
    at map[r, 0] + o map[r, 1] + c, so no packing copies run around the transposes.
      send (to rank q: its y columns of my planes)   block q = (N_t, nz, ny_q, n_1)
      recv (from rank r: my y columns of its planes) block r = (N_t, nz_r, ny, n_1)"""

    def __init__(self, layout, backend, group=None):
        import numpy as np
        self.layout, self.backend, self.group = layout, backend, group
        L = layout
        self.t1 = backend.empty(L.n_own)
        self.t2 = backend.empty(L.n_own)
        self.send = backend.empty(L.n_own)
        self.blk = backend.empty(L.n_blk)
        self.blk2 = backend.empty(L.n_blk)
        # all-to-all splits: to rank q go my planes x its y columns; from rank r come its planes x my columns
        self.split_own = [L.nt * L.nz * (L.ys[q + 1] - L.ys[q]) * L.n1 for q in range(L.world)]
        self.split_blk = [L.nt * (L.zs[r + 1] - L.zs[r]) * L.ny * L.n1 for r in range(L.world)]
        # direction-2 map over y (outer o = t nz + z, inner c = x) into the send layout
        ms = np.zeros((L.n2, 2), dtype=np.int64)
        off = 0
        for q in range(L.world):
            y0, y1 = L.ys[q], L.ys[q + 1]
            ms[y0:y1, 0] = off + (np.arange(y0, y1) - y0) * L.n1
            ms[y0:y1, 1] = (y1 - y0) * L.n1
            off += self.split_own[q]
        # direction-3 map over z (outer o = t, inner c = y' n_1 + x) into the receive layout
        mr = np.zeros((L.n3, 2), dtype=np.int64)
        off = 0
        for r in range(L.world):
            z0, z1 = L.zs[r], L.zs[r + 1]
            mr[z0:z1, 0] = off + (np.arange(z0, z1) - z0) * L.ny * L.n1
            mr[z0:z1, 1] = (z1 - z0) * L.ny * L.n1
            off += self.split_blk[r]
        self.map_send = backend.index_map(ms)
        self.map_recv = backend.index_map(mr)

    def apply_device(self, r_own, z_own):
        L, be = self.layout, self.backend
        # forward: U_1^T (contiguous), U_2^T (stride n_1) on the owned planes
        be.pc_mode(0, False, r_own, self.t1, L.nt * L.nz * L.n2, 1)
        if L.world == 1:
            # one rank: the owned slab already is the y-slab (no transposes)
            be.pc_mode(1, False, self.t1, self.t2, L.nt * L.nz, L.n1)
            be.pc_mode(2, False, self.t2, self.blk2, L.nt, L.ny * L.n1)
            be.pc_time_yslab(self.blk2, L.y_lo, L.y_hi)
            be.pc_mode(2, True, self.blk2, self.t2, L.nt, L.ny * L.n1)
            be.pc_mode(1, True, self.t2, self.t1, L.nt * L.nz, L.n1)
            be.pc_mode(0, True, self.t1, z_own, L.nt * L.nz * L.n2, 1)
            return
        be.pc_mode(1, False, self.t1, self.send, L.nt * L.nz, L.n1, omap=self.map_send)
        _all_to_all(self.blk2, self.send, self.split_blk, self.split_own, group=self.group)
        # y-slab: U_3^T (stride ny n_1) from the receive layout, time stage in place, U_3 back into it
        be.pc_mode(2, False, self.blk2, self.blk, L.nt, L.ny * L.n1, imap=self.map_recv)
        be.pc_time_yslab(self.blk, L.y_lo, L.y_hi)
        be.pc_mode(2, True, self.blk, self.blk2, L.nt, L.ny * L.n1, omap=self.map_recv)
        _all_to_all(self.send, self.blk2, self.split_own, self.split_blk, group=self.group)
        be.pc_mode(1, True, self.send, self.t2, L.nt * L.nz, L.n1, imap=self.map_send)
        be.pc_mode(0, True, self.t2, z_own, L.nt * L.nz * L.n2, 1)


def allreduce_sum(group=None):
    def red(t):
        if _staged(t, group):
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return red


def sharded_gmres(op, pc, ops, b_own, tol=1e-8, max_iter=200, group=None, log_path=None):
    """CGS2 GMRES on the owned slabs with all_reduce'd dot products."""
    return gmres_core(op.apply_device, pc.apply_device, ops, b_own, None, tol, max_iter,
                      allreduce=allreduce_sum(group), log_path=log_path)


# --------------------------------------------------------------------------
# CUDA backend
# --------------------------------------------------------------------------

class DeviceSlabBackend:
    """Local CUDA contexts of one rank: the z-slab operator and the preconditioner stages
    (libmonoiga_b200).  ``u``, ``w`` (variant B) are input-slab vectors."""

    def __init__(self, layout, space_time, final_time, capacitance, diffusion, constants,
                 stabilization=None, u=None, w=None, device=0, precond=None, op_context=None, lift=None,
                 iterate_is_zero=None):
        """``precond`` / ``op_context``: reuse a preconditioner and an operator context (the sharded
        fixed-point driver rebuilds only the operator's tables every sweep); ``lift``: u0 lifting
        coefficients of the input slab; ``iterate_is_zero``: the global zero-iterate decision."""
        from . import _lib
        from .operator import KroneckerOperator
        from .precond import FastDiagPreconditioner
        if len(space_time.spatial) != 3:
            raise ValueError("the space-sharded solve needs d = 3")
        self._lib = _lib
        L = layout
        self.op = KroneckerOperator(space_time, final_time, capacitance, diffusion, constants,
                                    u=u, w=w, stabilization=stabilization, device=device,
                                    z_planes=(L.z_lo, L.z_hi), context=op_context, lift=lift,
                                    iterate_is_zero=iterate_is_zero)
        self.pc = precond if precond is not None else FastDiagPreconditioner.build(
            space_time, final_time, capacitance, diffusion, constants["a"] * constants["c1"], device=device)
        self.device = self.op.ctx.device
        self.vec_ops = DeviceVecOps(self.op.ctx)

    def empty(self, n):
        return torch.empty(n, dtype=torch.float64, device=self.device)

    def apply_in(self, x_in, y_own):
        self.op.apply_device(x_in, y_own)

    def index_map(self, m):
        """(n, 2) int64 addressing map of mi_pc_mode_mapped, on the device."""
        return torch.from_numpy(m).to(self.device).contiguous()

    def pc_mode(self, l, inverse, src, dst, outer, inner, imap=None, omap=None):
        from .device import dptr
        self.pc.ctx.bind_stream()
        if imap is None and omap is None:
            self._lib.call("mi_pc_mode", self.pc.ctx.handle, l, 1 if inverse else 0, dptr(src), dptr(dst),
                           int(outer), int(inner))
        else:
            self._lib.call("mi_pc_mode_mapped", self.pc.ctx.handle, l, 1 if inverse else 0, dptr(src), dptr(dst),
                           int(outer), int(inner), None if imap is None else dptr(imap),
                           None if omap is None else dptr(omap))

    def pc_time_yslab(self, blk, y_lo, y_hi):
        from .device import dptr
        self.pc.ctx.bind_stream()
        self._lib.call("mi_pc_apply_time_yslab", self.pc.ctx.handle, dptr(blk), int(y_lo), int(y_hi))


# --------------------------------------------------------------------------
# Sharded fixed-point driver
# --------------------------------------------------------------------------

def gather_slabs(L, own, group=None):
    """The global (N_t, n_3, n_2 n_1) vector from every rank's owned z slab (all-gather, padded to the
    largest slab)."""
    world = L.world
    if world == 1:
        return own.clone()
    nmax = max(L.nt * (L.zs[r + 1] - L.zs[r]) * L.plane for r in range(world))
    dev = "cpu" if _staged(own, group) else own.device
    buf = torch.zeros(nmax, dtype=own.dtype, device=dev)
    buf[:own.numel()].copy_(own)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    full = torch.empty(L.nt, L.n3, L.plane, dtype=own.dtype, device=own.device)
    for r in range(world):
        z0, z1 = L.zs[r], L.zs[r + 1]
        n = L.nt * (z1 - z0) * L.plane
        full[:, z0:z1].copy_(parts[r][:n].view(L.nt, z1 - z0, L.plane))
    return full.view(-1)


def input_slab(L, full):
    """This rank's operator input slab (owned planes + halo planes) of a global vector."""
    v = full.view(L.nt, L.n3, L.plane)[:, L.z_lo - L.h_lo:L.z_hi + L.h_hi]
    return v.contiguous().view(-1)


def own_slab(L, full):
    return full.view(L.nt, L.n3, L.plane)[:, L.z_lo:L.z_hi].contiguous().view(-1)


def sharded_fixed_point_solve(problem, config=None, group=None, device=0):
    """fixed_point_solve (solver.py:239-386) with its hot path sharded over the ranks of ``group``.

    The potential solve of every sweep -- the z-slab operator (p-plane halo exchange), P^-1 with its
    two all-to-all transposes and GMRES with all-reduced CGS2 dots -- runs on each rank's z slab.  The
    per-sweep setup that needs the global iterate (the residual indicator, its low-rank split and the
    stencil tables, solver.py:291-324) and the recovery solve (a banded time solve and spatial mass
    solves, linalg.py:502-547) run replicated on every rank from all-gathered iterates; the load
    vector and the lifting are computed once.  Box geometries, d = 3, every-sweep or no indicator.
    Returns the same SolveResult on every rank (u, w gathered)."""
    import time as _time

    import numpy as np

    from .krylov import DeviceVecOps
    from .operator import KroneckerOperator, Stabilization
    from .precond import FastDiagPreconditioner
    from .problem import FixedPointConfig, FixedPointDiverged, SolveResult, box_of, lift_coefficients, load_vector
    from .theta import DeviceIndicator
    from .wsolve import RecoverySolver
    from .device import DeviceContext

    if config is None:
        config = FixedPointConfig()
    st = problem.space
    if len(st.spatial) != 3:
        raise ValueError("the sharded driver needs d = 3")
    if config.stabilization == "spline_upwind" and config.indicator_update != "every_sweep":
        raise NotImplementedError("the sharded driver recomputes the indicator every sweep")
    if config.linear_solver == "direct":
        raise NotImplementedError("the direct (host LU) linear solver is not part of the device path")
    t0 = _time.perf_counter()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = torch.device("cuda", device)
    p = st.spatial[0].degree
    L = ZSlabLayout(st.num_time, [s.dimension for s in st.spatial], p, rank, world)
    Lb, _ = box_of(problem.geometry)
    T, consts = problem.final_time, problem.reaction_constants()
    D = problem.D if np.atleast_1d(problem.D).size > 1 else problem.scalar_D()
    # replicated, once: load vector, lifting, recovery solver and its mass operator, indicator
    f = load_vector(st, problem.geometry, problem.source, device=device)
    f = (f if torch.is_tensor(f) else torch.from_numpy(np.ascontiguousarray(f))).to(dev)
    f_own = own_slab(L, f)
    lift_np = lift_coefficients(problem)
    lift = None if lift_np is None else torch.from_numpy(lift_np).to(dev)
    lift_in = None
    if lift is not None:
        lift_in = lift.view(L.n3, L.plane)[L.z_lo - L.h_lo:L.z_hi + L.h_hi].contiguous().view(-1)
    mass_op = KroneckerOperator(st, T, 0.0, 0.0, {"c1": 1.0, "a": 1.0, "c2": 0.0}, lengths=Lb, device=device,
                                lift=lift, lift_in_reaction=False)
    g_lift = mass_op.lift_apply() if lift is not None else None
    wsolver = RecoverySolver(st, T, problem.b, problem.d_e, config.linear_tol, lengths=Lb, device=device)
    indicator = DeviceIndicator(problem, device) if config.stabilization == "spline_upwind" else None
    # sharded, once: the preconditioner; the operator context is reused by every sweep
    pc = FastDiagPreconditioner.build(st, T, problem.C_m, D, problem.a * problem.c1, lengths=Lb, device=device)
    op_ctx = DeviceContext(st, device, zslab=(L.z_lo, L.z_hi, L.h_lo, L.h_hi))
    def allmax(v):
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if _staged(f_own, group) else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return float(t.item())

    u_own = torch.zeros(L.n_own, dtype=torch.float64, device=dev)
    w_own = torch.zeros_like(u_own)
    increments, gmres_iters, pcg_iters = [], [], []
    ind_vals = None
    frozen_stab = None
    alpha = config.relaxation
    for k in range(1, config.max_iterations + 1):
        u_full = gather_slabs(L, u_own, group)
        w_full = gather_slabs(L, w_own, group)
        zero = allmax(float(u_own.abs().max().item()) + float(w_own.abs().max().item())) == 0.0
        stab = None
        if indicator is not None:
            if frozen_stab is not None:
                stab = frozen_stab
            else:
                fresh = indicator.compute(u_full, w_full, on_device=True, lift=lift).values
                fresh = torch.as_tensor(fresh, device=dev)
                freeze = False
                if ind_vals is not None and alpha < 1.0:
                    drift = float((fresh - ind_vals).abs().max().item())
                    fresh = alpha * fresh + (1.0 - alpha) * ind_vals
                    if config.indicator_freeze_tol > 0.0 and k > 1 and drift * alpha <= config.indicator_freeze_tol:
                        freeze = True
                ind_vals = fresh
                stab = Stabilization(st, ind_vals, config.lowrank_tol, problem.C_m, lengths=Lb)
                if freeze:
                    frozen_stab = stab
        be = DeviceSlabBackend(L, st, T, problem.C_m, D, consts, stabilization=stab,
                               u=None if zero else input_slab(L, u_full), w=None if zero else input_slab(L, w_full),
                               device=device, precond=pc, op_context=op_ctx, lift=lift_in, iterate_is_zero=zero)
        sop, spc = ShardedOperator(L, be, group), ShardedPreconditioner(L, be, group)
        rhs = f_own if lift is None else f_own - be.op.lift_apply()
        u_t, nit, _ = sharded_gmres(sop, spc, be.vec_ops, rhs, tol=config.linear_tol, max_iter=st.num_dof,
                                    group=group)
        gmres_iters.append(nit)
        if config.evolve_recovery:
            g_full = mass_op.matvec(u_full)
            if g_lift is not None:
                g_full = g_full + g_lift
            w_t_full, w_its = wsolver.solve(problem.b * g_full)
            pcg_iters.extend(w_its)
            w_t = own_slab(L, w_t_full)
        else:
            w_t = w_own
        u_new = alpha * u_t + (1.0 - alpha) * u_own
        w_new = alpha * w_t + (1.0 - alpha) * w_own
        inc = allmax(float((u_new - u_own).abs().max().item()))
        increments.append(inc)
        u_own, w_own = u_new, w_new
        if inc <= config.tolerance:
            u_full = gather_slabs(L, u_own, group).cpu().numpy()
            w_full = gather_slabs(L, w_own, group).cpu().numpy()
            return SolveResult(u_full, w_full, k, increments, True, gmres_iters, pcg_iters,
                               _time.perf_counter() - t0, None, {}, lift_np)
    result = SolveResult(gather_slabs(L, u_own, group).cpu().numpy(), gather_slabs(L, w_own, group).cpu().numpy(),
                         config.max_iterations, increments, False, gmres_iters, pcg_iters,
                         _time.perf_counter() - t0, None, {}, lift_np)
    raise FixedPointDiverged("fixed point did not reach %.2e in %d iterations"
                             % (config.tolerance, config.max_iterations), result)
