"""Interface field from the 1D periodic field equation (poisson.py:1-60).

``solve_field`` runs on the device (libpk ``pk_field``): prefix sum in
np.cumsum order plus the zero-mean gauge, with the reference's solvability
guard raised as :class:`SolvabilityViolation`.
"""

from __future__ import annotations

import numpy as np

from .engine import Device
from .mesh import PhaseMesh

SOLVABILITY_RTOL = 1e-10  # poisson.py:18


def solve_field(rho, rho_bar: float, mesh: PhaseMesh, rtol: float | None = None) -> np.ndarray:
    rho = np.asarray(rho, dtype=float)
    if rho.shape != (mesh.nx,):
        raise ValueError(f"expected shape ({mesh.nx},), got {rho.shape}")
    rtol = SOLVABILITY_RTOL if rtol is None else rtol
    dev = Device.for_mesh(mesh)
    r = dev.t(rho.reshape(1, -1))
    E = dev.scratch("field_E", (1, mesh.nx))
    dev.field(r, dev.t(np.array([float(rho_bar)])), E, rtol)
    dev.check()
    return E[0].cpu().numpy().copy()


def gauss_residual(E, rho, rho_bar, mesh: PhaseMesh) -> float:
    """Max-norm residual of the discrete relation (host diagnostic, poisson.py:57-60)."""
    lhs = (E - np.roll(E, 1)) / mesh.dx
    return float(np.max(np.abs(lhs - (rho - rho_bar))))
