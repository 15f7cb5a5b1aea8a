"""Time-sharded solve over torch.distributed: one process per GPU.

Each rank owns a contiguous slab of time rows [t_lo, t_hi) of every
(N_t, N_s) vector.  The exchanges are exactly the ones the path needs:

* operator A: a p_t-row halo of x from each time neighbour (send/recv), then
  the local stencil + time-filter kernel on the extended slab; only the
  owned rows of the result are kept.  (The reaction's time elements reach
  p_t rows as well, so the same halo covers it; u, w halos are exchanged
  once when the operator is built.)
* preconditioner P^-1: spatial transforms on the owned rows, an all-to-all
  transpose to spatial-column slabs (every rank then holds all N_t rows of
  N_s/G eigen-columns), the time stage (Q^T, arrowhead, Q) locally, the
  inverse all-to-all, inverse spatial transforms.
* GMRES: the CGS2 dot products and norms are summed with all_reduce; the
  Hessenberg recurrence is replicated on every rank (krylov.gmres_core).

The orchestration is backend-agnostic: ``DeviceSlabBackend`` runs the CUDA
kernels of libmonoiga_b200 (NCCL on the GPU box); the CPU tests plug in a
reference backend with the gloo process group (tests/test_sharded_cpu.py).
"""

import numpy as np
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


class SlabLayout:
    """Row / column ownership of one rank."""

    def __init__(self, nt, ns, halo, rank, world):
        if nt < world * max(halo, 1):
            raise ValueError("too few time rows (%d) for %d ranks with halo %d" % (nt, world, halo))
        self.nt, self.ns, self.halo, self.rank, self.world = nt, ns, halo, rank, world
        self.rows = split(nt, world)
        self.cols = split(ns, world)
        self.t_lo, self.t_hi = self.rows[rank], self.rows[rank + 1]
        self.e_lo = max(0, self.t_lo - halo)
        self.e_hi = min(nt, self.t_hi + halo)
        self.s_lo, self.s_hi = self.cols[rank], self.cols[rank + 1]

    @property
    def nown(self):
        return self.t_hi - self.t_lo

    @property
    def next_(self):
        return self.e_hi - self.e_lo

    @property
    def ncols(self):
        return self.s_hi - self.s_lo


def exchange_halo(layout, x_own, x_ext, group=None):
    """x_ext[rows e_lo..e_hi) <- own rows + halos from the time neighbours."""
    L, ns = layout, layout.ns
    off = (L.t_lo - L.e_lo) * ns
    x_ext[off:off + L.nown * ns].copy_(x_own)
    ops = []
    left, right = L.rank - 1, L.rank + 1
    hl = L.t_lo - L.e_lo                      # rows received from the left neighbour
    hr = L.e_hi - L.t_hi                      # rows received from the right neighbour
    nsend = min(L.halo, L.nown)
    if left >= 0:
        # my first rows are the left neighbour's right halo; its last rows are my left halo
        ops.append(dist.P2POp(dist.isend, x_ext[off:off + nsend * ns], left, group))
        ops.append(dist.P2POp(dist.irecv, x_ext[:hl * ns], left, group))
    if right < L.world:
        ops.append(dist.P2POp(dist.isend, x_ext[off + (L.nown - nsend) * ns:off + L.nown * ns], right, group))
        ops.append(dist.P2POp(dist.irecv, x_ext[off + L.nown * ns:off + (L.nown + hr) * ns], right, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return x_ext


class ShardedOperator:
    """y_own = (A x)_own with a p_t-row halo exchange (``apply_device``)."""

    def __init__(self, layout, backend, group=None):
        self.layout, self.backend, self.group = layout, backend, group
        n = layout.next_ * layout.ns
        self.x_ext = backend.empty(n)
        self.y_ext = backend.empty(n)

    def apply_device(self, x_own, y_own):
        L = self.layout
        exchange_halo(L, x_own, self.x_ext, self.group)
        self.backend.apply_ext(self.x_ext, self.y_ext)
        off = (L.t_lo - L.e_lo) * L.ns
        y_own.copy_(self.y_ext[off:off + L.nown * L.ns])


class ShardedPreconditioner:
    """z_own = (P^-1 r)_own with two all-to-all transposes (``apply_device``)."""

    def __init__(self, layout, backend, group=None):
        self.layout, self.backend, self.group = layout, backend, group
        L = layout
        self.s_own = backend.empty(L.nown * L.ns)
        self.send = backend.empty(L.nown * L.ns)
        self.blk = backend.empty(L.nt * L.ncols)
        self.in_splits = [L.nown * (L.cols[r + 1] - L.cols[r]) for r in range(L.world)]
        self.out_splits = [(L.rows[r + 1] - L.rows[r]) * L.ncols for r in range(L.world)]

    def apply_device(self, r_own, z_own):
        L, be = self.layout, self.backend
        be.pc_spatial(r_own, self.s_own, L.nown, inverse=False)
        # pack: for each destination rank, (own rows x its columns), contiguous
        S = self.s_own.view(L.nown, L.ns)
        off = 0
        for q in range(L.world):
            c0, c1 = L.cols[q], L.cols[q + 1]
            self.send[off:off + L.nown * (c1 - c0)].view(L.nown, c1 - c0).copy_(S[:, c0:c1])
            off += L.nown * (c1 - c0)
        if L.world > 1:
            dist.all_to_all_single(self.blk, self.send, self.out_splits, self.in_splits, group=self.group)
        else:
            self.blk.copy_(self.send)
        # blk is the time-major (N_t x ncols) block of my eigen-columns
        be.pc_time(self.blk, L.ncols, L.s_lo)
        if L.world > 1:
            dist.all_to_all_single(self.send, self.blk, self.in_splits, self.out_splits, group=self.group)
        else:
            self.send.copy_(self.blk)
        off = 0
        for q in range(L.world):
            c0, c1 = L.cols[q], L.cols[q + 1]
            S[:, c0:c1].copy_(self.send[off:off + L.nown * (c1 - c0)].view(L.nown, c1 - c0))
            off += L.nown * (c1 - c0)
        be.pc_spatial(self.s_own, z_own, L.nown, inverse=True)


def allreduce_sum(group=None):
    def red(t):
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
    """Local CUDA contexts of one rank: the extended-slab operator and the
    preconditioner stages (libmonoiga_b200)."""

    def __init__(self, layout, space_time, final_time, capacitance, diffusion, constants,
                 stabilization=None, u=None, w=None, device=0):
        from . import _lib
        from .device import DeviceContext
        from .operator import KroneckerOperator
        from .precond import FastDiagPreconditioner
        self._lib = _lib
        L = layout
        self.op = KroneckerOperator(space_time, final_time, capacitance, diffusion, constants,
                                    u=u, w=w, stabilization=stabilization, device=device,
                                    time_rows=(L.e_lo, L.e_hi))
        self.pc = FastDiagPreconditioner.build(space_time, final_time, capacitance, diffusion,
                                               constants["a"] * constants["c1"], device=device)
        self.device = self.op.ctx.device
        self.vec_ops = DeviceVecOps(self.op.ctx)

    def empty(self, n):
        return torch.empty(n, dtype=torch.float64, device=self.device)

    def apply_ext(self, x_ext, y_ext):
        self.op.apply_device(x_ext, y_ext)

    def pc_spatial(self, src, dst, nrows, inverse):
        from .device import dptr
        self.pc.ctx.bind_stream()
        self._lib.call("mi_pc_apply_spatial", self.pc.ctx.handle, dptr(src), dptr(dst), nrows,
                       1 if inverse else 0)

    def pc_time(self, blk, ncols, col0):
        from .device import dptr
        self.pc.ctx.bind_stream()
        self._lib.call("mi_pc_apply_time", self.pc.ctx.handle, dptr(blk), ncols, col0)
