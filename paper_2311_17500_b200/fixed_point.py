"""Relaxed fixed-point driver on the device (drop-in for the reference's
``fixed_point_solve``, solver.py:239-386).

Each sweep freezes the Rogers-McCulloch reaction at the previous iterate,
solves the potential system with the device GMRES + fast-diagonalisation
preconditioner (the hot path), solves the recovery system with the device
w-solve, relaxes both, and stops when max |u_new - u| <= tolerance.
Spline Upwind: the indicator is recomputed on the device (DeviceIndicator,
the reference compute_theta) and relaxed/frozen exactly as
solver.py:291-324 does, then factorised and turned into device stencil
channels.
"""

import time as _time

import numpy as np
import torch

from .device import DeviceContext
from .krylov import gmres
from .operator import KroneckerOperator, Stabilization
from .precond import FastDiagPreconditioner
from .problem import (FixedPointConfig, FixedPointDiverged, GaussGrid, SolveResult, box_of, lift_coefficients,
                      load_vector)
from .theta import DeviceIndicator, MappedDeviceIndicator
from .wsolve import RecoverySolver


class _Workspace:
    """solver.py:163-211 (box geometry, device objects)."""

    def __init__(self, problem, config, device=0):
        from .geometry import MappedSpatialData, is_mapped
        st = problem.space
        if config.linear_solver == "direct":
            raise NotImplementedError("the direct (host LU) linear solver is not part of the device path")
        # mapped geometries: quadrature M_s / K_s, |det J| reaction, separable-weight P^-1 (solver.py:167-202)
        from .geometry import is_fibre
        fibre = problem.D if is_fibre(problem.D) else None
        self.sd = (MappedSpatialData(st.spatial, problem.geometry, conductivity=fibre,
                                     coefficient_rank=config.coefficient_rank, coefficient_tol=config.coefficient_tol)
                   if is_mapped(problem.geometry) else None)
        self.L = None if self.sd is not None else box_of(problem.geometry)[0]
        self.device = device
        self.indicator = None
        if config.stabilization == "spline_upwind":
            self.indicator = (DeviceIndicator(problem, device) if self.sd is None else
                              MappedDeviceIndicator(problem, device,
                                                    grid=GaussGrid(st, problem.geometry, mapped=self.sd)))
        if self.indicator is not None and self.sd is not None:
            self.grid = self.indicator._grid
            self.f_vec = load_vector(st, problem.geometry, problem.source, self.grid, device=device)
        elif self.indicator is not None and problem.source is not None:
            # one host evaluation of the source feeds both the load vector and the indicator's
            # device-resident copy
            self.grid = self.indicator._grid = GaussGrid(st, problem.geometry, mapped=self.sd)
            self.f_vec = load_vector(st, problem.geometry, problem.source, self.grid,
                                     chunks=self.indicator.source_chunks(problem.source))
        else:
            self.grid = GaussGrid(st, problem.geometry, mapped=self.sd)
            self.f_vec = load_vector(st, problem.geometry, problem.source, self.grid, device=device)
        self.pc_ctx = DeviceContext(st, device)
        self.precond = FastDiagPreconditioner.build(st, problem.final_time, problem.C_m, problem.scalar_D(),
                                                    problem.a * problem.c1, lengths=self.L, context=self.pc_ctx,
                                                    spatial_data=self.sd)
        # u0 lifting (DESIGN 7): the lifted slab's coefficients stay on the device for every sweep
        lift = lift_coefficients(problem)
        self.lift = None if lift is None else torch.from_numpy(lift).to(torch.device("cuda", device))
        # M_t (x) M_s for g = b (M_t (x) M_s) u  (C_m = D = 0, unit reaction: channel c1 = M_t (x) M_s);
        # with a lift, g also takes the lifted column b (T M[1:, 0] (x) M_s) u0
        self.mass_op = KroneckerOperator(st, problem.final_time, 0.0, 0.0, {"c1": 1.0, "a": 1.0, "c2": 0.0},
                                         lengths=self.L, device=device, spatial_data=self.sd, lift=self.lift,
                                         lift_in_reaction=False)
        self.g_lift = self.mass_op.lift_apply() if self.lift is not None else None
        self.wsolver = RecoverySolver(st, problem.final_time, problem.b, problem.d_e, config.linear_tol,
                                      lengths=self.L, device=device, spatial_data=self.sd)

    def operator(self, problem, u_k, w_k, stab):
        # one operator context for all sweeps: its buffers are reused (dalloc keeps large-enough
        # allocations), so a sweep rebuilds tables, not allocations
        if getattr(self, "op_ctx", None) is None:
            self.op_ctx = DeviceContext(problem.space, self.device)
        return KroneckerOperator(problem.space, problem.final_time, problem.C_m, problem.scalar_D(),
                                 problem.reaction_constants(), u=u_k, w=w_k, stabilization=stab,
                                 lengths=self.L, device=self.device, context=self.op_ctx, spatial_data=self.sd,
                                 lift=self.lift)


def _host_indicator(ind):
    """SolveResult carries a numpy indicator (the driver may hold it on the device)."""
    v = getattr(ind, "values", None)
    if torch.is_tensor(v):
        ind.values = v.cpu().numpy()
    return ind


def _indicator_values(ind):
    v = ind if torch.is_tensor(ind) else getattr(ind, "values", ind)
    return v if torch.is_tensor(v) else np.asarray(v, float)


class _Phases:
    """Wall time per driver phase (synchronised, so GPU work is attributed to its phase)."""

    def __init__(self):
        self.sec = {}
        self._t = None

    def start(self):
        torch.cuda.synchronize()
        self._t = _time.perf_counter()

    def stop(self, name):
        torch.cuda.synchronize()
        self.sec[name] = self.sec.get(name, 0.0) + _time.perf_counter() - self._t


def fixed_point_solve(problem, config=None, device=0):
    """solver.py:239-386 on the device; returns SolveResult (numpy u, w)."""
    if config is None:
        config = FixedPointConfig()
    st = problem.space
    t0 = _time.perf_counter()
    ph = _Phases()

    frozen_stab = None
    galerkin_sweeps = 0
    frozen_indicator = None
    if config.stabilization == "spline_upwind" and config.indicator_update == "frozen":
        from dataclasses import replace
        pre = fixed_point_solve(problem, replace(config, stabilization="off"), device)
        galerkin_sweeps = pre.iterations
        if config.indicator_override is not None:
            frozen_indicator = config.indicator_override(problem, pre.u, pre.w)
        else:
            from .geometry import is_mapped
            cls = MappedDeviceIndicator if is_mapped(problem.geometry) else DeviceIndicator
            frozen_indicator = cls(problem, device).compute(pre.u, pre.w, lift=pre.lift)
        from .geometry import is_mapped
        frozen_stab = Stabilization(st, _indicator_values(frozen_indicator), config.lowrank_tol, problem.C_m,
                                    lengths=None if is_mapped(problem.geometry) else box_of(problem.geometry)[0])

    ph.start()
    ws = _Workspace(problem, config, device)
    # the iterate stays on the device between sweeps; only the result comes back to the host
    dev = ws.pc_ctx.device
    f_dev = (ws.f_vec.to(dev) if torch.is_tensor(ws.f_vec)
             else torch.from_numpy(np.ascontiguousarray(ws.f_vec)).to(dev))
    ph.stop("setup")
    lift_host = None if ws.lift is None else ws.lift.cpu().numpy()
    u = torch.zeros(st.num_dof, dtype=torch.float64, device=dev)
    w = torch.zeros_like(u)
    increments, gmres_iters, pcg_iters = [], [], []
    indicator = frozen_indicator
    alpha = config.relaxation
    freeze_now = False

    for k in range(galerkin_sweeps + 1, galerkin_sweeps + config.max_iterations + 1):
        stab = None
        if config.stabilization == "spline_upwind":
            if frozen_stab is not None:
                stab = frozen_stab
            else:
                ph.start()
                if config.indicator_override is not None:
                    fresh = config.indicator_override(problem, u.cpu().numpy(), w.cpu().numpy())
                else:
                    fresh = ws.indicator.compute(u, w, on_device=True, lift=ws.lift)
                ph.stop("indicator")
                if indicator is not None and alpha < 1.0:
                    prev = _indicator_values(indicator)
                    fv = _indicator_values(fresh)
                    if torch.is_tensor(fv) or torch.is_tensor(prev):
                        fv, prev = (torch.as_tensor(v, device=dev) for v in (fv, prev))
                        drift = float((fv - prev).abs().max().item())
                    else:
                        drift = float(np.max(np.abs(fv - prev)))
                    fresh.values = alpha * fv + (1.0 - alpha) * prev
                    if (config.indicator_freeze_tol > 0.0 and k > galerkin_sweeps + 1
                            and drift * alpha <= config.indicator_freeze_tol):
                        freeze_now = True
                indicator = fresh
                ph.start()
                stab = Stabilization(st, _indicator_values(indicator), config.lowrank_tol, problem.C_m,
                                     lengths=ws.L)
                ph.stop("stabilization")
                if freeze_now:
                    frozen_stab = stab
        ph.start()
        op = ws.operator(problem, u, w, stab)
        ph.stop("operator_setup")
        ph.start()
        rhs = f_dev if ws.lift is None else f_dev - op.lift_apply()
        u_tilde, nit, _ = gmres(op, rhs, precond=ws.precond, tol=config.linear_tol)
        ph.stop("gmres")
        gmres_iters.append(nit)

        ph.start()
        if config.evolve_recovery:
            g_vec = ws.mass_op.matvec(u)
            if ws.g_lift is not None:
                g_vec = g_vec + ws.g_lift
            g_vec = problem.b * g_vec
            w_tilde, w_its = ws.wsolver.solve(g_vec)
            pcg_iters.extend(w_its)
        else:
            w_tilde = w
        ph.stop("w_solve")

        u_new = alpha * u_tilde + (1.0 - alpha) * u
        w_new = alpha * w_tilde + (1.0 - alpha) * w
        inc = float((u_new - u).abs().max().item())
        increments.append(inc)
        if config.verbose:
            print("  sweep %3d: increment %.3e" % (k, inc))
        u, w = u_new, w_new
        if inc <= config.tolerance:
            return SolveResult(u.cpu().numpy(), w.cpu().numpy(), k, increments, True, gmres_iters, pcg_iters,
                               _time.perf_counter() - t0, _host_indicator(indicator), ph.sec, lift_host)
    result = SolveResult(u.cpu().numpy(), w.cpu().numpy(), galerkin_sweeps + config.max_iterations, increments,
                         False, gmres_iters, pcg_iters, _time.perf_counter() - t0, _host_indicator(indicator), ph.sec,
                         lift_host)
    raise FixedPointDiverged("fixed point did not reach %.2e in %d iterations"
                             % (config.tolerance, config.max_iterations), result)
