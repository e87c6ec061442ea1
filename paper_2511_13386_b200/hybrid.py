"""Spatially hybrid stepper S^HMM (hybrid.py:1-226) on the device.

``hybrid_propagate`` is one launch of the persistent fine-propagator kernel
(libpk ``pk_fine_propagate``): labels, flips, lifts, the masked micro-macro
update and both field solves of every step stay on the GPU; the host only
forms the step schedule and the scalar constants.  With ``trace`` the
reference's per-substep callback is honoured on a slow path (one launch per
step, state copied back each step).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .adaptation import DomainLabels, Thresholds
from .engine import Device, HybridKnobs, make_phase
from .fluid import substep_sizes
from .kinetic import KineticStepParams, Workspace  # noqa: F401
from .mesh import MacroState, MicroState, PhaseMesh
from .poisson import SOLVABILITY_RTOL


@dataclass(frozen=True)
class HybridOptions:
    adaptation: bool = True
    combine: str = "or"
    scale_remainder: bool = False
    reinit: str = "lift"
    lift_order: int = 2
    time_elim: str = "leading"


@dataclass(frozen=True)
class HybridState:
    macro: MacroState
    micro: MicroState
    labels: DomainLabels
    E_prev: np.ndarray

    @classmethod
    def initial(cls, macro: MacroState, micro: MicroState, mesh: PhaseMesh) -> "HybridState":
        return cls(macro=macro, micro=micro, labels=DomainLabels.all_kinetic(mesh.nx),
                   E_prev=macro.E)


def knobs_of(opts: HybridOptions | None, th: Thresholds | None) -> HybridKnobs:
    if opts is None or not opts.adaptation:
        return HybridKnobs(adaptation=False)
    if opts.combine not in ("or", "and"):
        raise ValueError(f"combine must be 'or' or 'and', got {opts.combine!r}")
    return HybridKnobs(adaptation=True, combine=opts.combine,
                       scale_remainder=opts.scale_remainder, reinit=opts.reinit,
                       lift_order=opts.lift_order, time_elim=opts.time_elim,
                       delta0=th.delta0, eta0=th.eta0)


def _device_run(mesh: PhaseMesh, rho, g, E, E_prev, labels, eps, sched, th, opts, rho_bar,
                field_rtol, init_flags=0):
    """Run one slice through ``sched = [(n_full, dt), (n_rem, rem)]`` on the device."""
    dev = Device.for_mesh(mesh)
    nx, nv = mesh.nx, mesh.nv
    sched = list(sched) + [(0, sched[0][1])] * (2 - len(sched))
    phases = [make_phase(mesh, [eps], [dt], [n]) for n, dt in sched]
    knobs = knobs_of(opts, th)
    rtol = SOLVABILITY_RTOL if field_rtol is None else field_rtol
    rho_d = dev.t(np.asarray(rho, dtype=float).reshape(1, nx).copy())
    E_d = dev.t(np.asarray(E if E is not None else np.zeros(nx), dtype=float).reshape(1, nx).copy())
    Ep_d = dev.t(np.asarray(E_prev if E_prev is not None else np.zeros(nx),
                            dtype=float).reshape(1, nx).copy())
    if labels is None:
        kc = np.ones(nx, dtype=np.uint8)
        ki = kc.copy()
    else:
        kc = labels.kinetic_cells.astype(np.uint8)
        ki = labels.kinetic_ifaces.astype(np.uint8)
    kc_d, ki_d = dev.t(kc.reshape(1, nx).copy()), dev.t(ki.reshape(1, nx).copy())
    g_d = dev.t(np.asarray(g, dtype=float).reshape(1, nx, nv).copy())
    rb = dev.t(np.array([float(rho_bar)]))
    dev.fine(rho_d, E_d, Ep_d, kc_d, ki_d, g_d, rb, [init_flags], phases, knobs, [eps], rtol)
    dev.check()
    return dict(rho=rho_d[0].cpu().numpy(), E=E_d[0].cpu().numpy(),
                E_prev=Ep_d[0].cpu().numpy(),
                kc=kc_d[0].cpu().numpy().astype(bool), ki=ki_d[0].cpu().numpy().astype(bool),
                g=g_d[0].cpu().numpy().reshape((nx,) + mesh.vgrid.shape))


def hybrid_step(state: HybridState, p: KineticStepParams, th: Thresholds, opts: HybridOptions,
                mesh: PhaseMesh, rho_bar: float, dt: float | None = None, ws=None,
                field_rtol: float | None = None) -> HybridState:
    """One hybrid step (hybrid.py:123-188)."""
    dt = p.dt if dt is None else dt
    p.check(dt, mesh)
    out = _device_run(mesh, state.macro.rho, state.micro.g, state.macro.E, state.E_prev,
                      state.labels, p.eps, [(1, dt)], th, opts, rho_bar, field_rtol)
    return HybridState(
        macro=MacroState(rho=out["rho"], E=out["E"], t=state.macro.t + dt),
        micro=MicroState(g=out["g"]),
        labels=DomainLabels(kinetic_cells=out["kc"], kinetic_ifaces=out["ki"]),
        E_prev=out["E_prev"])


def hybrid_propagate(state: HybridState, t_end: float, p: KineticStepParams, th: Thresholds,
                     opts: HybridOptions, mesh: PhaseMesh, rho_bar: float,
                     trace: Callable[[HybridState], None] | None = None,
                     field_rtol: float | None = None) -> HybridState:
    """Advance to exactly t_end (hybrid.py:191-226)."""
    n_full, rem = substep_sizes(state.macro.t, t_end, p.dt)
    if n_full == 0 and rem == 0.0:
        return HybridState(macro=MacroState(rho=state.macro.rho, E=state.macro.E, t=t_end),
                           micro=state.micro, labels=state.labels, E_prev=state.E_prev)
    if trace is not None:
        cur = state
        for h in [p.dt] * n_full + ([rem] if rem > 0.0 else []):
            cur = hybrid_step(cur, p, th, opts, mesh, rho_bar, dt=h, field_rtol=field_rtol)
            trace(cur)
        return HybridState(macro=MacroState(rho=cur.macro.rho, E=cur.macro.E, t=t_end),
                           micro=cur.micro, labels=cur.labels, E_prev=cur.E_prev)
    if n_full > 0:
        p.check(p.dt, mesh)
    if rem > 0.0:
        p.check(rem, mesh)
    out = _device_run(mesh, state.macro.rho, state.micro.g, state.macro.E, state.E_prev,
                      state.labels, p.eps,
                      [(n_full, p.dt), (1 if rem > 0.0 else 0, rem if rem > 0.0 else p.dt)],
                      th, opts, rho_bar, field_rtol)
    return HybridState(
        macro=MacroState(rho=out["rho"], E=out["E"], t=t_end),
        micro=MicroState(g=out["g"]),
        labels=DomainLabels(kinetic_cells=out["kc"], kinetic_ifaces=out["ki"]),
        E_prev=out["E_prev"])
