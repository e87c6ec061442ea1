"""Chapman-Enskog lifting (lifting.py:1-110), on the device (libpk ``pk_lift``:
one CTA per slice for the O(nx) stencil scalars, one warp per interface row
for the velocity polynomial and the two zero-mass projections)."""

from __future__ import annotations

import numpy as np

from .engine import Device
from .errors import MeshTooSmall
from .mesh import MicroState, PhaseMesh

LIFT_ORDERS = (1, 2)
DEFAULT_ORDER = 2


def lift(rho, E, eps, mesh: PhaseMesh, order: int = DEFAULT_ORDER, dE_dt=None,
         time_elim: str = "leading", rho_bar: float | None = None, project: bool = True,
         ws=None) -> MicroState:
    if order not in LIFT_ORDERS:
        raise ValueError(f"lift order must be one of {LIFT_ORDERS}, got {order}")
    if mesh.nx < 7:
        raise MeshTooSmall(f"lifting stencils need nx >= 7, got {mesh.nx}")
    if order >= 2:
        if time_elim == "higher_order":
            if rho_bar is None:
                raise ValueError("higher_order elimination needs rho_bar")
        elif time_elim != "leading":
            raise ValueError(
                f"time_elim must be 'leading' or 'higher_order', got {time_elim!r}")
    dev = Device.for_mesh(mesh)
    nx, nv = mesh.nx, mesh.nv
    r = dev.t(np.asarray(rho, dtype=float).reshape(1, nx))
    e = dev.t(np.asarray(E, dtype=float).reshape(1, nx))
    de = None if dE_dt is None else dev.t(np.asarray(dE_dt, dtype=float).reshape(1, nx))
    rb = dev.t(np.array([0.0 if rho_bar is None else float(rho_bar)]))
    g = dev.scratch("lift_g", (1, nx, nv))
    dev.lift(r, e, de, rb, [eps], order, time_elim if order >= 2 else "leading", project, g)
    dev.check()
    return MicroState(g=g[0].cpu().numpy().reshape((nx,) + mesh.vgrid.shape).copy())


def project_zero_mass(g, mesh: PhaseMesh):
    """In-place two-pass projection (host helper, lifting.py:97-105)."""
    for _ in range(2):
        b = mesh.bracket_x(g) / mesh.vgrid.m0
        g -= b[..., None, None, None] * mesh.vgrid.M
    return g


def mass_defect(g, mesh: PhaseMesh):
    """Per-interface <g> (host diagnostic, lifting.py:108-110)."""
    return mesh.bracket_x(g)
