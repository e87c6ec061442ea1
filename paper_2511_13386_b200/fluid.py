"""Explicit drift-diffusion scheme S0: the coarse propagator G and the
fluid-cell update (fluid.py:1-118).  Propagation runs on the device
(libpk ``pk_coarse_chain``, one CTA per chain, state in shared memory)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .engine import Device
from .errors import StabilityViolation
from .mesh import MacroState, PhaseMesh
from .poisson import SOLVABILITY_RTOL

CFL_SAFETY = 0.9
_BOUND_SLACK = 1.0 + 1e-12


@dataclass(frozen=True)
class FluidStepParams:
    dt: float
    m2: float

    @classmethod
    def default(cls, mesh: PhaseMesh, cfl_safety: float = CFL_SAFETY) -> "FluidStepParams":
        m2 = mesh.vgrid.m2
        return cls(dt=cfl_safety * mesh.dx**2 / (2.0 * m2), m2=m2)

    def check(self, dt: float, mesh: PhaseMesh) -> None:
        bound = mesh.dx**2 / (2.0 * self.m2)
        if dt > bound * _BOUND_SLACK:
            raise StabilityViolation(
                f"dt={dt:.6e} exceeds parabolic bound dx^2/(2 m2)={bound:.6e}")


def substep_sizes(t0: float, t_end: float, dt: float):
    """fluid.py:80-92."""
    span = t_end - t0
    if span < 0.0:
        raise ValueError(f"t_end={t_end} earlier than state time {t0}")
    if span == 0.0:
        return 0, 0.0
    n_full = int(np.floor(span / dt + 1e-12))
    rem = span - n_full * dt
    if rem <= 1e-12 * max(span, dt):
        rem = 0.0
    return n_full, rem


def fluid_flux(rho, E, mesh: PhaseMesh):
    """Host O(nx) helper (fluid.py:48-52); the device computes J inside F and G."""
    rho_next = np.roll(rho, -1)
    return (rho_next - rho) / mesh.dx - E * 0.5 * (rho + rho_next)


def _rho_update(rho, J, m2, dt, mesh: PhaseMesh):
    """Host O(nx) helper (fluid.py:55-57)."""
    return rho + m2 * (dt / mesh.dx) * (J - np.roll(J, 1))


def _run_chain(mesh, rho_rows, E_in, nfull, rem, dt, rho_bar, rtol, m2):
    dev = Device.for_mesh(mesh)
    nchain = rho_rows.shape[0]
    r = dev.t(np.ascontiguousarray(rho_rows, dtype=float))
    out = dev.scratch("chain_out", (nchain, 1, mesh.nx))
    Eo = dev.scratch("chain_E", (nchain, mesh.nx))
    dev.chain(r, out, None, Eo, None, [nfull] * nchain, [rem] * nchain, dt,
              dev.t(np.full(nchain, float(rho_bar))), rtol,
              E_in=None if E_in is None else dev.t(np.ascontiguousarray(E_in, dtype=float)), m2=m2)
    dev.check()
    return out[:, 0].cpu().numpy().copy(), Eo.cpu().numpy().copy()


def fluid_step(state: MacroState, p: FluidStepParams, mesh: PhaseMesh, rho_bar: float,
               dt: float | None = None, refresh_field: bool = True,
               field_rtol: float | None = None) -> MacroState:
    """One explicit step with the caller's field (fluid.py:60-77)."""
    dt = p.dt if dt is None else dt
    p.check(dt, mesh)
    rtol = (SOLVABILITY_RTOL if field_rtol is None else field_rtol) if refresh_field else np.inf
    rho, E = _run_chain(mesh, np.asarray(state.rho)[None], np.asarray(state.E)[None], 0, dt, dt,
                        rho_bar, rtol, p.m2)
    return MacroState(rho=rho[0], E=E[0] if refresh_field else state.E, t=state.t + dt)


def fluid_propagate(state: MacroState, t_end: float, p: FluidStepParams, mesh: PhaseMesh,
                    rho_bar: float, field_rtol: float | None = None) -> MacroState:
    """Advance to exactly t_end (fluid.py:95-118)."""
    n_full, rem = substep_sizes(state.t, t_end, p.dt)
    if n_full == 0 and rem == 0.0:
        return MacroState(rho=state.rho, E=state.E, t=t_end)
    if n_full > 0:
        p.check(p.dt, mesh)
    if rem > 0.0:
        p.check(rem, mesh)
    rtol = SOLVABILITY_RTOL if field_rtol is None else field_rtol
    rho, E = _run_chain(mesh, np.asarray(state.rho)[None], None, n_full, rem, p.dt, rho_bar, rtol,
                        p.m2)
    return MacroState(rho=rho[0], E=E[0], t=t_end)
