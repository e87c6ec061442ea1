"""Relaxed AP micro-macro scheme S^MM (kinetic.py:1-298).

Step-size rules and relaxation constants are host arithmetic (as in the
reference); every step of g and rho runs on the device in the persistent
fine-propagator kernel (libpk ``pk_fine_propagate`` with adaptation off,
which is the all-kinetic path of the hybrid stepper).

eps may be a float (the reference) or an :class:`EpsProfile` (the eps(x)
extension): per-interface relaxation constants and the
conservative density update ``rho_i -= dt/dx (flux_i/eps_i - flux_{i-1}/eps_{i-1})``,
which reduces bitwise to the reference where eps is constant.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .engine import relaxation_coefficients  # noqa: F401  (re-export)
from .errors import StabilityViolation
from .mesh import MacroState, MicroState, PhaseMesh

_BOUND_SLACK = 1.0 + 1e-12
UPWIND_ORDER = 1


@dataclass(frozen=True, eq=False)
class EpsProfile:
    """Spatially varying Knudsen number: eps at interfaces and at cells."""

    iface: np.ndarray
    cell: np.ndarray

    def __post_init__(self):
        if np.any(np.asarray(self.iface) <= 0.0) or np.any(np.asarray(self.cell) <= 0.0):
            raise ValueError("eps must be positive")

    @staticmethod
    def from_function(fn, mesh: PhaseMesh) -> "EpsProfile":
        return EpsProfile(np.asarray(fn(mesh.x_interfaces), dtype=float),
                          np.asarray(fn(mesh.x_centers), dtype=float))

    def distinct(self):
        return sorted(set(self.iface.tolist()) | set(self.cell.tolist()))


def eps_values(eps):
    return eps.distinct() if isinstance(eps, EpsProfile) else [float(eps)]


class Workspace:
    """Accepted for signature compatibility (kinetic.py:36-48); device scratch
    is owned by the libpk context."""

    def buf(self, key, shape):
        return np.empty(shape)


@dataclass(frozen=True)
class KineticStepParams:
    eps: object
    dt: float

    def __post_init__(self):
        if not isinstance(self.eps, EpsProfile) and self.eps <= 0.0:
            raise ValueError("eps must be positive")

    @classmethod
    def default(cls, mesh: PhaseMesh, eps, e_max: float = 0.0, cfl_safety: float = 0.9,
                transport_theta: float = 0.9) -> "KineticStepParams":
        dt = stable_dt(mesh, eps, e_max=e_max, cfl_safety=cfl_safety, theta=transport_theta)
        return cls(eps=eps, dt=dt)

    def check(self, dt: float, mesh: PhaseMesh) -> None:
        parabolic = mesh.dx**2 / (2.0 * mesh.vgrid.m2)
        transport = mesh.dx / mesh.v_star
        if dt > parabolic * _BOUND_SLACK or dt > transport * _BOUND_SLACK:
            raise StabilityViolation(
                f"dt={dt:.6e} exceeds stability bounds "
                f"(parabolic {parabolic:.6e}, transport {transport:.6e})")
        # the same scalar rule per distinct eps; an eps(x) profile has thousands
        # of values and every parareal window re-checks the same (eps, dt):
        # the first offending value (or None) is memoised
        lam = _lambda_transport(mesh, 0.0)
        key = (_eps_key(self.eps), dt, lam)
        hit = _CHECKS.get(key)
        if hit is None or hit[0] is not self.eps:
            bad = None
            for e in eps_values(self.eps):
                if _transport_amplification(dt, e, lam) > 1.0 + 1e-9:
                    bad = e
                    break
            hit = _CHECKS[key] = (self.eps, bad)
            while len(_CHECKS) > 256:
                _CHECKS.pop(next(iter(_CHECKS)))
        if hit[1] is not None:
            raise StabilityViolation(
                f"dt={dt:.6e} violates the relaxed transport condition at eps={hit[1]:g}")


_CHECKS: dict = {}    # (eps, dt, lambda) -> (eps, first offending eps or None)
_STABLE: dict = {}    # (eps, mesh constants, knobs) -> (eps, dt)


def _eps_key(eps):
    return ("profile", id(eps)) if isinstance(eps, EpsProfile) else float(eps)


def _lambda_transport(mesh: PhaseMesh, e_max: float) -> float:
    lam = 2.0 * mesh.v_star / mesh.dx
    if e_max > 0.0:
        lam += 2.0 * e_max / mesh.vgrid.dvx
    return lam


def _transport_amplification(dt: float, eps: float, lam: float) -> float:
    z = dt / eps**2
    return eps * (-np.expm1(-z)) * lam / (1.0 + np.exp(-z))


def _stable_dt_scalar(mesh, eps, e_max, cfl_safety, theta, transport_safety):
    dt_max = min(cfl_safety * mesh.dx**2 / (2.0 * mesh.vgrid.m2),
                 transport_safety * mesh.dx / mesh.v_star)
    lam = _lambda_transport(mesh, e_max)
    if _transport_amplification(dt_max, eps, lam) <= theta:
        return dt_max
    lo, hi = 0.0, dt_max
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if _transport_amplification(mid, eps, lam) <= theta:
            lo = mid
        else:
            hi = mid
    return lo


def stable_dt(mesh: PhaseMesh, eps, e_max: float = 0.0, cfl_safety: float = 0.9,
              theta: float = 0.9, transport_safety: float = 0.5) -> float:
    """kinetic.py:107-138; for an EpsProfile the minimum over its values
    (memoised per profile: the same scalar bisection per distinct value)."""
    key = (_eps_key(eps), mesh.dx, mesh.v_star, mesh.vgrid.m2, mesh.vgrid.dvx, float(e_max),
           cfl_safety, theta, transport_safety)
    hit = _STABLE.get(key)
    if hit is None or hit[0] is not eps:
        dt = min(_stable_dt_scalar(mesh, e, e_max, cfl_safety, theta, transport_safety)
                 for e in eps_values(eps))
        hit = _STABLE[key] = (eps, dt)
        while len(_STABLE) > 256:
            _STABLE.pop(next(iter(_STABLE)))
    return hit[1]


def kinetic_step(state, p: KineticStepParams, mesh: PhaseMesh, rho_bar: float,
                 dt: float | None = None, ws=None):
    """One full step (kinetic.py:255-273)."""
    from .hybrid import _device_run

    dt = p.dt if dt is None else dt
    p.check(dt, mesh)
    macro, micro = state
    out = _device_run(mesh, macro.rho, micro.g, macro.E, None, None, p.eps, [(1, dt)],
                      None, None, rho_bar, None)
    return MacroState(rho=out["rho"], E=out["E"], t=macro.t + dt), MicroState(g=out["g"])


def kinetic_propagate(state, t_end: float, p: KineticStepParams, mesh: PhaseMesh,
                      rho_bar: float):
    """Advance to exactly t_end (kinetic.py:276-298)."""
    from .fluid import substep_sizes
    from .hybrid import _device_run

    macro, micro = state
    n_full, rem = substep_sizes(macro.t, t_end, p.dt)
    if n_full == 0 and rem == 0.0:
        return MacroState(rho=macro.rho, E=macro.E, t=t_end), micro
    if n_full > 0:
        p.check(p.dt, mesh)
    if rem > 0.0:
        p.check(rem, mesh)
    out = _device_run(mesh, macro.rho, micro.g, macro.E, None, None, p.eps,
                      [(n_full, p.dt), (1 if rem > 0.0 else 0, rem if rem > 0.0 else p.dt)],
                      None, None, rho_bar, None)
    return MacroState(rho=out["rho"], E=out["E"], t=t_end), MicroState(g=out["g"])
