"""numpy restatement of the parakin fine propagator (1D-x / 1D-v), TEST ORACLE.

Every function cites the reference lines it restates (paths relative to
``/root/reference/pkg/src/parakin``).  Arrays: ``g`` is ``(nx, nv)`` (the
reference's ``(nx, nvx, 1, 1)`` with the unit axes dropped — SURVEY F3 shows
the reduction is exact), per-x arrays are ``(nx,)``.

Bit-exactness rules followed throughout:
  * velocity integrals fold mirror pairs, then numpy pairwise-sum the folded
    row (``ndarray.sum`` along the contiguous last axis);
  * the field uses a sequential ``np.cumsum`` and pairwise sums;
  * elementwise expressions keep the reference's evaluation order;
  * scalar constants (kappa1/2, eps**2, dt/(eps dx), dx**-p) are formed with
    Python floats exactly as the reference forms them.

eps(x) extension: wherever the reference takes a scalar
``eps`` this module also accepts an :class:`EpsProfile` (eps at interfaces and
at cells).  Interface quantities use ``eps_if[i]``; the conservative density
update uses ``c_i = dt/(eps_i dx)`` and, where ``c_i == c_{i-1}``, the
reference's factored form ``c*(flux_i - flux_{i-1})`` so that a constant
profile reproduces the reference bitwise.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

TWO_PI = 2.0 * np.pi
SOLVABILITY_RTOL = 1e-10          # poisson.py:18
ADAPTIVE_FIELD_RTOL = 1e-5        # parareal.py:48
CFL_SAFETY = 0.9                  # fluid.py:23
_SLACK = 1.0 + 1e-12              # fluid.py:25, kinetic.py:22

STENCILS = {                      # adaptation.py:29-34
    1: (-1 / 60, 3 / 20, -3 / 4, 0.0, 3 / 4, -3 / 20, 1 / 60),
    2: (1 / 90, -3 / 20, 3 / 2, -49 / 18, 3 / 2, -3 / 20, 1 / 90),
    3: (1 / 8, -1.0, 13 / 8, 0.0, -13 / 8, 1.0, -1 / 8),
    4: (-1 / 6, 2.0, -13 / 2, 28 / 3, -13 / 2, 2.0, -1 / 6),
}


class OracleError(Exception):
    """Base of the oracle's error taxonomy (mirrors errors.py:4-26)."""


class OracleSolvability(OracleError):
    pass


class OracleStability(OracleError):
    pass


class OracleNonFinite(OracleError):
    pass


# ---------------------------------------------------------------------------
# phase mesh (mesh.py)


@dataclass(frozen=True)
class Grid1V:
    nx: int
    nv: int
    x_star: float
    v_star: float
    dx: float
    dvx: float
    dv3: float
    vx: np.ndarray
    M: np.ndarray
    m0: float
    m2: float
    xi_plus: np.ndarray = field(repr=False)
    xi_minus: np.ndarray = field(repr=False)
    xi_M: np.ndarray = field(repr=False)
    x_centers: np.ndarray = field(repr=False)
    x_interfaces: np.ndarray = field(repr=False)


def centers(n: int, v_star: float) -> np.ndarray:
    """mesh.py:36-44 — mirrored cell centres."""
    dv = 2.0 * v_star / n
    half = (np.arange(n // 2) + 0.5) * dv
    if n % 2 == 0:
        return np.concatenate([-half[::-1], half])
    inner = (np.arange(n // 2) + 1.0) * dv
    return np.concatenate([-inner[::-1], [0.0], inner])


def vsum(q: np.ndarray, dv3: float) -> np.ndarray:
    """mesh.py:95-109,124-133 — folded velocity integral over the last axis."""
    n = q.shape[-1]
    h = n // 2
    folded = q[..., :h] + q[..., ::-1][..., :h]
    total = folded.sum(axis=-1)
    if n % 2 == 1:
        total = total + q[..., h]
    return total * dv3


def vsum_scalar(q: np.ndarray, dv3: float) -> float:
    """mesh.py:112-121 — the whole-array bracket (one velocity row)."""
    n = q.shape[0]
    h = n // 2
    total = (q[:h] + q[::-1][:h]).sum()
    if n % 2 == 1:
        total = total + q[h]
    return float(total * dv3)


def make_grid(nx: int, nv: int, x_star: float = TWO_PI, v_star: float = 8.0) -> Grid1V:
    """mesh.py:197-236 with nvy = nvz = 1 (MeshSpec.validate bypassed)."""
    vx = centers(nv, v_star)
    dvx = 2.0 * v_star / nv
    dvy = 2.0 * v_star / 1
    dv3 = dvx * dvy * dvy
    v_sq = vx**2 + 0.0**2 + 0.0**2
    M = np.exp(-0.5 * v_sq) / TWO_PI**1.5
    for _ in range(2):
        M = M / vsum_scalar(M, dv3)
    m0 = vsum_scalar(M, dv3)
    m2 = vsum_scalar(vx**2 * M, dv3)
    dx = x_star / nx
    return Grid1V(
        nx=nx, nv=nv, x_star=x_star, v_star=v_star, dx=dx, dvx=dvx, dv3=dv3,
        vx=vx, M=M, m0=m0, m2=m2,
        xi_plus=np.maximum(vx, 0.0), xi_minus=np.minimum(vx, 0.0), xi_M=vx * M,
        x_centers=(np.arange(nx) + 0.5) * dx,
        x_interfaces=(np.arange(nx) + 1.0) * dx,
    )


def prev_(a):
    return np.roll(a, 1, axis=0)


def next_(a):
    return np.roll(a, -1, axis=0)


def to_cells(q):
    """mesh.py:187-190."""
    return 0.5 * (prev_(q) + q)


def to_ifaces(q):
    """mesh.py:192-194."""
    return 0.5 * (q + next_(q))


# ---------------------------------------------------------------------------
# eps(x) extension


@dataclass(frozen=True)
class EpsProfile:
    """eps sampled at interfaces x_{i+1/2} (``iface``) and centres (``cell``)."""

    iface: np.ndarray
    cell: np.ndarray

    @staticmethod
    def constant(eps: float, nx: int) -> "EpsProfile":
        return EpsProfile(np.full(nx, float(eps)), np.full(nx, float(eps)))

    @staticmethod
    def from_function(fn, grid: Grid1V) -> "EpsProfile":
        return EpsProfile(np.asarray(fn(grid.x_interfaces), dtype=float),
                          np.asarray(fn(grid.x_centers), dtype=float))

    def distinct(self):
        return sorted(set(float(e) for e in self.iface) | set(float(e) for e in self.cell))


def per_iface(eps, nx, fn):
    """Apply the scalar rule ``fn(eps_value)`` per interface (one call per
    distinct value, so constants are formed exactly like the reference)."""
    if isinstance(eps, EpsProfile):
        cache = {}
        out = np.empty(nx)
        for i, e in enumerate(eps.iface):
            e = float(e)
            if e not in cache:
                cache[e] = fn(e)
            out[i] = cache[e]
        return out
    return fn(float(eps))


def per_cell(eps, nx, fn):
    if isinstance(eps, EpsProfile):
        cache = {}
        out = np.empty(nx)
        for i, e in enumerate(eps.cell):
            e = float(e)
            if e not in cache:
                cache[e] = fn(e)
            out[i] = cache[e]
        return out
    return fn(float(eps))


def eps_values(eps):
    return eps.distinct() if isinstance(eps, EpsProfile) else [float(eps)]


# ---------------------------------------------------------------------------
# field (poisson.py)


def field(rho, rho_bar, grid: Grid1V, rtol=None):
    """poisson.py:21-54 — prefix sum + zero-mean gauge with solvability guard."""
    rho = np.asarray(rho, dtype=float)
    rtol = SOLVABILITY_RTOL if rtol is None else rtol
    src = (rho - rho_bar) * grid.dx
    defect = src.sum()
    scale = np.abs(rho).sum() * grid.dx
    if abs(defect) > rtol * max(scale, np.finfo(float).tiny):
        raise OracleSolvability(f"net source {defect:.3e} exceeds {rtol:.0e} * {scale:.3e}")
    src -= defect / grid.nx
    E = np.cumsum(src)
    E -= E.mean()
    return E


# ---------------------------------------------------------------------------
# drift-diffusion limit (fluid.py)


def flux_J(rho, E, grid: Grid1V):
    """fluid.py:48-52."""
    rn = next_(rho)
    return (rn - rho) / grid.dx - E * 0.5 * (rho + rn)


def rho_fluid(rho, J, m2, dt, grid: Grid1V):
    """fluid.py:55-57."""
    return rho + m2 * (dt / grid.dx) * (J - prev_(J))


def fluid_dt(grid: Grid1V, cfl=CFL_SAFETY) -> float:
    """fluid.py:35-38."""
    return cfl * grid.dx**2 / (2.0 * grid.m2)


def fluid_check(dt, grid: Grid1V):
    """fluid.py:40-46."""
    bound = grid.dx**2 / (2.0 * grid.m2)
    if dt > bound * _SLACK:
        raise OracleStability(f"dt={dt:.6e} exceeds parabolic bound {bound:.6e}")


def schedule(t0, t_end, dt):
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


def fluid_advance(rho, t0, t_end, dt, grid: Grid1V, rho_bar, rtol=None):
    """fluid.py:60-77,95-118.  Returns (rho, E)."""
    n_full, rem = schedule(t0, t_end, dt)
    if n_full == 0 and rem == 0.0:
        return rho, None
    E = field(rho, rho_bar, grid, rtol)
    for h in [dt] * n_full + ([rem] if rem > 0.0 else []):
        fluid_check(h, grid)
        J = flux_J(rho, E, grid)
        rho = rho_fluid(rho, J, grid.m2, h, grid)
        E = field(rho, rho_bar, grid, rtol)
    return rho, E


# ---------------------------------------------------------------------------
# micro-macro AP scheme (kinetic.py)


def _lam(grid: Grid1V, e_max):
    """kinetic.py:91-97."""
    lam = 2.0 * grid.v_star / grid.dx
    if e_max > 0.0:
        lam += 2.0 * e_max / grid.dvx
    return lam


def _amp(dt, eps, lam):
    """kinetic.py:100-104."""
    z = dt / eps**2
    return eps * (-np.expm1(-z)) * lam / (1.0 + np.exp(-z))


def stable_dt_scalar(grid: Grid1V, eps, e_max=0.0, cfl=0.9, theta=0.9, tsafe=0.5):
    """kinetic.py:107-138."""
    dt_max = min(cfl * grid.dx**2 / (2.0 * grid.m2), tsafe * grid.dx / grid.v_star)
    lam = _lam(grid, e_max)
    if _amp(dt_max, eps, lam) <= theta:
        return dt_max
    lo, hi = 0.0, dt_max
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if _amp(mid, eps, lam) <= theta:
            lo = mid
        else:
            hi = mid
    return lo


def stable_dt(grid: Grid1V, eps, e_max=0.0):
    """kinetic.py:107-138; eps(x): the minimum over the distinct eps values."""
    return min(stable_dt_scalar(grid, e, e_max) for e in eps_values(eps))


def kinetic_check(dt, eps, grid: Grid1V):
    """kinetic.py:77-88 (every distinct eps for a profile)."""
    parabolic = grid.dx**2 / (2.0 * grid.m2)
    transport = grid.dx / grid.v_star
    if dt > parabolic * _SLACK or dt > transport * _SLACK:
        raise OracleStability(f"dt={dt:.6e} exceeds stability bounds")
    for e in eps_values(eps):
        if _amp(dt, e, _lam(grid, 0.0)) > 1.0 + 1e-9:
            raise OracleStability(f"dt={dt:.6e} violates the relaxed transport condition at eps={e:g}")


def kappas(dt, eps_value: float):
    """kinetic.py:141-145."""
    z = dt / eps_value**2
    return float(np.exp(-z)), float(eps_value * (-np.expm1(-z)))


def kappa_rows(dt, eps, nx):
    """(kappa1, kappa2) broadcastable against g rows."""
    k1 = per_iface(eps, nx, lambda e: kappas(dt, e)[0])
    k2 = per_iface(eps, nx, lambda e: kappas(dt, e)[1])
    if isinstance(eps, EpsProfile):
        return k1[:, None], k2[:, None]
    return k1, k2


def transport(g, E, grid: Grid1V, bmask=None):
    """kinetic.py:148-194 (``bmask``: hybrid.py:103-105 projection mask)."""
    out = grid.xi_plus * (g - prev_(g))
    out += grid.xi_minus * (next_(g) - g)
    out /= grid.dx
    Ep = (np.maximum(E, 0.0) / grid.dvx)[:, None]
    Em = (np.minimum(E, 0.0) / grid.dvx)[:, None]
    dm = np.empty_like(g)
    dm[:, 0] = g[:, 0]
    dm[:, 1:] = g[:, 1:] - g[:, :-1]
    out += dm * Ep
    dp = np.empty_like(g)
    dp[:, :-1] = g[:, 1:] - g[:, :-1]
    dp[:, -1] = -g[:, -1]
    out += dp * Em
    b = vsum(grid.vx * g, grid.dv3)
    if bmask is not None:
        b = np.where(bmask, b, 0.0)
    dc = (next_(b) - prev_(b)) / (2.0 * grid.dx)
    out -= grid.M * dc[:, None]
    return out


def micro(g, rho, E, dt, eps, grid: Grid1V, bmask=None):
    """kinetic.py:210-224 / hybrid.py:91-110."""
    k1, k2 = kappa_rows(dt, eps, grid.nx)
    J = flux_J(rho, E, grid)
    forcing = transport(g, E, grid, bmask) + grid.xi_M * J[:, None]
    return k1 * g - k2 * forcing


def rho_kinetic(rho, flux, eps, dt, grid: Grid1V):
    """kinetic.py:232-240; eps(x): conservative split form (module doc)."""
    if not isinstance(eps, EpsProfile):
        return rho - (dt / (eps * grid.dx)) * (flux - prev_(flux))
    c = per_iface(eps, grid.nx, lambda e: dt / (e * grid.dx))
    cp = prev_(c)
    same = c == cp
    factored = c * (flux - prev_(flux))
    split = c * flux - cp * prev_(flux)
    return rho - np.where(same, factored, split)


def kinetic_advance(rho, g, t0, t_end, dt, eps, grid: Grid1V, rho_bar):
    """kinetic.py:255-298.  Returns (rho, E, g); E is None for an empty span."""
    n_full, rem = schedule(t0, t_end, dt)
    E = None
    for h in [dt] * n_full + ([rem] if rem > 0.0 else []):
        kinetic_check(h, eps, grid)
        E = field(rho, rho_bar, grid)
        g = micro(g, rho, E, h, eps, grid)
        rho = rho_kinetic(rho, vsum(grid.vx * g, grid.dv3), eps, h, grid)
        E = field(rho, rho_bar, grid)
    return rho, E, g


def kinetic_steps(rho, g, n, dt, eps, grid: Grid1V, rho_bar):
    """n plain ``kinetic_step`` calls (kinetic.py:255-273)."""
    E = None
    for _ in range(n):
        kinetic_check(dt, eps, grid)
        E = field(rho, rho_bar, grid)
        g = micro(g, rho, E, dt, eps, grid)
        rho = rho_kinetic(rho, vsum(grid.vx * g, grid.dv3), eps, dt, grid)
        E = field(rho, rho_bar, grid)
    return rho, E, g


# ---------------------------------------------------------------------------
# adaptation (adaptation.py)


def stencil(values, order, dx):
    """adaptation.py:65-77."""
    out = np.zeros_like(values, dtype=float)
    for c, o in zip(STENCILS[order], (-3, -2, -1, 0, 1, 2, 3)):
        if c != 0.0:
            out += c * np.roll(values, -o)
    return out * dx ** (-order)


def remainder_fields(rho, E, dtE_c, rho_bar, grid: Grid1V):
    """adaptation.py:120-138."""
    dx = grid.dx
    J_c = to_cells(flux_J(rho, E, grid))
    E_c = to_cells(E)
    d1J = stencil(J_c, 1, dx)
    d2J = stencil(J_c, 2, dx)
    d3J = stencil(J_c, 3, dx)
    d1r = stencil(rho, 1, dx)
    return -d3J + E_c * d2J + (2.0 * rho - 3.0 * rho_bar) * d1J + 2.0 * J_c * d1r - d1r * dtE_c


def remainder(rho, E, E_prev, dt, rho_bar, grid: Grid1V):
    """adaptation.py:141-152."""
    return remainder_fields(rho, E, to_cells((E - E_prev) / dt), rho_bar, grid)


def gnorm(g, grid: Grid1V):
    """adaptation.py:155-159."""
    sq = vsum(g * g, grid.dv3)
    return np.sqrt(0.5 * (prev_(sq) + sq))


def labels_from(R, gn, delta0, eta0, combine="or"):
    """adaptation.py:162-181 + DomainLabels.from_cells (100-105)."""
    fR = np.abs(R) < delta0
    fg = gn < eta0
    if combine == "or":
        fluid = fR | fg
    elif combine == "and":
        fluid = fR & fg
    else:
        raise ValueError(f"combine must be 'or' or 'and', got {combine!r}")
    kc = ~fluid
    return kc, kc | np.roll(kc, -1)


# ---------------------------------------------------------------------------
# Chapman-Enskog lift (lifting.py)


def lift(rho, E, eps, grid: Grid1V, order=2, dE_dt=None, time_elim="leading",
         rho_bar=None, project=True):
    """lifting.py:38-105 (eps(x): per-interface eps)."""
    if order not in (1, 2):
        raise ValueError(f"lift order must be one of (1, 2), got {order}")
    nx = grid.nx
    J = flux_J(rho, E, grid)
    neg = per_iface(eps, nx, lambda e: -e)
    g = grid.xi_M * (neg * J)[:, None]
    if order >= 2:
        dJ = to_ifaces(stencil(to_cells(J), 1, grid.dx))
        drift = dJ - E * J
        if time_elim == "higher_order":
            if rho_bar is None:
                raise ValueError("higher_order elimination needs rho_bar")
            dtE_c = to_cells(dE_dt) if dE_dt is not None else np.zeros(nx)
            R_if = to_ifaces(remainder_fields(rho, E, dtE_c, rho_bar, grid))
        elif time_elim == "leading":
            R_if = None
        else:
            raise ValueError(f"time_elim must be 'leading' or 'higher_order', got {time_elim!r}")
        w = (grid.vx**2 - 1.0) * grid.M
        e2 = per_iface(eps, nx, lambda e: e**2)
        if isinstance(eps, EpsProfile):
            g += (e2[:, None] * w) * drift[:, None]
            if R_if is not None:
                g += (e2[:, None] * grid.M) * R_if[:, None]
        else:
            g += (e2 * w) * drift[:, None]
            if R_if is not None:
                g += (e2 * grid.M) * R_if[:, None]
    g = g.copy()
    if project:
        for _ in range(2):
            b = vsum(g, grid.dv3) / grid.m0
            g -= b[:, None] * grid.M
    return g


# ---------------------------------------------------------------------------
# hybrid stepper (hybrid.py)


@dataclass(frozen=True)
class HState:
    rho: np.ndarray
    E: np.ndarray
    g: np.ndarray
    kc: np.ndarray
    ki: np.ndarray
    E_prev: np.ndarray
    t: float

    @staticmethod
    def start(rho, E, g, t=0.0):
        """hybrid.py:68-72 — all kinetic, E_prev = E."""
        nx = rho.shape[0]
        ones = np.ones(nx, dtype=bool)
        return HState(rho, E, g, ones, ones.copy(), E, t)


@dataclass(frozen=True)
class HOpts:
    """hybrid.py:45-55."""

    adaptation: bool = True
    combine: str = "or"
    scale_remainder: bool = False
    reinit: str = "lift"
    lift_order: int = 2
    time_elim: str = "leading"


def hstep(st: HState, dt, eps, delta0, eta0, opts: HOpts, grid: Grid1V, rho_bar,
          rtol=None) -> HState:
    """hybrid.py:123-188, with the three dispatch paths written as one masked
    update (hybrid.py:75-120; SURVEY F17 shows the equivalence)."""
    kinetic_check(dt, eps, grid)
    rho, g = st.rho, st.g
    E = field(rho, rho_bar, grid, rtol)
    nx = grid.nx
    if opts.adaptation:
        R = remainder(rho, E, st.E_prev, dt, rho_bar, grid)
        if opts.scale_remainder:
            R = per_cell(eps, nx, lambda e: e**2) * R
        kc, ki = labels_from(R, gnorm(g, grid), delta0, eta0, opts.combine)
        flip = ki & ~st.ki
        if flip.any():
            g = g.copy()
            if opts.reinit == "lift":
                lifted = lift(rho, E, eps, grid, order=opts.lift_order,
                              dE_dt=(E - st.E_prev) / dt, time_elim=opts.time_elim,
                              rho_bar=rho_bar)
                g[flip] = lifted[flip]
            elif opts.reinit == "zero":
                g[flip] = 0.0
            else:
                raise ValueError(f"reinit must be 'lift' or 'zero', got {opts.reinit!r}")
    else:
        kc = np.ones(nx, dtype=bool)
        ki = kc.copy()
    if ki.any():
        gk = micro(g, rho, E, dt, eps, grid, bmask=ki)
        gk[~ki] = 0.0
        flux = np.where(ki, vsum(grid.vx * gk, grid.dv3), 0.0)
        rho_k = rho_kinetic(rho, flux, eps, dt, grid)
    else:
        gk = np.zeros_like(g)
        rho_k = rho
    rho_f = rho_fluid(rho, flux_J(rho, E, grid), grid.m2, dt, grid)
    rho_new = np.where(kc, rho_k, rho_f)
    E_new = field(rho_new, rho_bar, grid, rtol)
    return HState(rho_new, E_new, gk, kc, ki, E, st.t + dt)


def hpropagate(st: HState, t_end, dt, eps, delta0, eta0, opts: HOpts, grid: Grid1V,
               rho_bar, rtol=None, trace=None) -> HState:
    """hybrid.py:191-226."""
    n_full, rem = schedule(st.t, t_end, dt)
    if n_full == 0 and rem == 0.0:
        return replace(st, t=t_end)
    for h in [dt] * n_full + ([rem] if rem > 0.0 else []):
        st = hstep(st, h, eps, delta0, eta0, opts, grid, rho_bar, rtol)
        if trace is not None:
            trace(st)
    return replace(st, t=t_end)


# ---------------------------------------------------------------------------
# parareal engine (parareal.py)


@dataclass(frozen=True)
class PConfig:
    """parareal.py:55-77 (eps may be an EpsProfile)."""

    eps: object
    t_final: float
    ng: int
    k_max: int = 50
    tol: float = 1e-10
    parareal_enabled: bool = True
    delta0: float = 1e-5
    eta0: float = 1e-5
    opts: HOpts = HOpts()

    @property
    def bounds(self):
        return np.linspace(0.0, self.t_final, self.ng + 1)

    @property
    def rtol(self):
        """parareal.py:51-52 (field_guard)."""
        return ADAPTIVE_FIELD_RTOL if self.opts.adaptation else None


def default_steps(cfg: PConfig, grid: Grid1V, E0):
    """parareal.py:138-146 -> (coarse dt, fine dt)."""
    return fluid_dt(grid), stable_dt(grid, cfg.eps, e_max=float(np.max(np.abs(E0))))


def fine_window(n, rho_in, g0, cfg: PConfig, dt_f, grid: Grid1V, rho_bar):
    """parareal.py:153-190 -> (rho_out, kinetic_fraction)."""
    b = cfg.bounds
    E = field(rho_in, rho_bar, grid, cfg.rtol)
    if n == 1:
        g = g0
    else:
        g = lift(rho_in, E, cfg.eps, grid, order=cfg.opts.lift_order,
                 time_elim=cfg.opts.time_elim, rho_bar=rho_bar)
    st = HState.start(rho_in, E, g, float(b[n - 1]))
    out = hpropagate(st, float(b[n]), dt_f, cfg.eps, cfg.delta0, cfg.eta0, cfg.opts,
                     grid, rho_bar, cfg.rtol)
    return out.rho, float(np.count_nonzero(out.kc)) / grid.nx


def coarse(rho_in, n, cfg: PConfig, dt_c, grid: Grid1V, rho_bar, rtol="cfg"):
    b = cfg.bounds
    rtol = cfg.rtol if rtol == "cfg" else rtol
    out, _ = fluid_advance(rho_in, float(b[n - 1]), float(b[n]), dt_c, grid, rho_bar, rtol)
    return out


@dataclass
class PResult:
    status: str
    iterations: int
    rows: list
    err: list
    kinetic_fraction: np.ndarray
    jumps: list

    @property
    def boundary_rho(self):
        return self.rows[-1]


def parareal(cfg: PConfig, rho0, g0, grid: Grid1V, rho_bar, fine=None) -> PResult:
    """parareal.py:210-353 (serial coordinator; windows in index order).
    ``fine`` overrides the fine window (the reference's ``_fine_window`` seam)."""
    fine = fine or fine_window
    E0 = field(rho0, rho_bar, grid)
    dt_c, dt_f = default_steps(cfg, grid, E0)
    ng = cfg.ng
    frac = np.zeros(ng + 1)
    if not cfg.parareal_enabled:
        # parareal.py:356-392: state carries across windows
        row = np.empty((ng + 1, grid.nx))
        row[0] = rho0
        st = HState.start(rho0, E0, g0, 0.0)
        for n in range(1, ng + 1):
            st = hpropagate(st, float(cfg.bounds[n]), dt_f, cfg.eps, cfg.delta0, cfg.eta0,
                            cfg.opts, grid, rho_bar, cfg.rtol)
            row[n] = st.rho
            frac[n] = float(np.count_nonzero(st.kc)) / grid.nx
        return PResult("serial", 0, [row], [], frac, [])
    # coarse sweep (parareal.py:210-229): default field guard, E carried
    row = np.empty((ng + 1, grid.nx))
    row[0] = rho0
    rho = rho0
    t = 0.0
    for n in range(1, ng + 1):
        rho, _ = fluid_advance(rho, t, float(cfg.bounds[n]), dt_c, grid, rho_bar, None)
        t = float(cfg.bounds[n])
        row[n] = rho
    rows = [row]
    errs, jumps = [], []
    status = "max_iterations"
    for k in range(cfg.k_max):
        row_k = rows[k]
        deltas = {}
        for n in range(k + 1, ng + 1):
            f_rho, kf = fine(n, row_k[n - 1], g0, cfg, dt_f, grid, rho_bar)
            deltas[n] = f_rho - coarse(row_k[n - 1], n, cfg, dt_c, grid, rho_bar)
            frac[n] = kf
        for n in range(k + 1, ng + 1):
            if not np.isfinite(deltas[n]).all():
                raise OracleNonFinite(f"non-finite jump in window {n}")
        new = row_k.copy()
        for n in range(k + 1, ng + 1):
            new[n] = coarse(new[n - 1], n, cfg, dt_c, grid, rho_bar) + deltas[n]
        if not np.isfinite(new).all():
            raise OracleNonFinite(f"non-finite density after iteration {k + 1}")
        err = float(np.max(np.abs(new - row_k)))
        rows.append(new)
        errs.append(err)
        jumps.append(deltas)
        if err < cfg.tol:
            status = "converged"
            break
    return PResult(status, len(errs), rows, errs, frac, jumps)


def lift_restart_chain(cfg: PConfig, rho0, g0, grid: Grid1V, rho_bar):
    """parareal.py:395-413."""
    E0 = field(rho0, rho_bar, grid)
    _, dt_f = default_steps(cfg, grid, E0)
    row = np.empty((cfg.ng + 1, grid.nx))
    row[0] = rho0
    for n in range(1, cfg.ng + 1):
        row[n], _ = fine_window(n, row[n - 1], g0, cfg, dt_f, grid, rho_bar)
    return row


# ---------------------------------------------------------------------------
# initial-data decomposition (experiment.py:64-85, recipe only)


def decompose(f_of_x, grid: Grid1V):
    """Split f(x, v) (a callable returning (len(x), nv)) into cell density,
    zero-mass interface perturbation and rho_bar, as experiment.py:70-79."""
    rho_cells = vsum(f_of_x(grid.x_centers), grid.dv3)
    f_if = f_of_x(grid.x_interfaces)
    rho_if = vsum(f_if, grid.dv3)
    g0 = f_if - rho_if[:, None] * grid.M
    rho_bar = float(rho_cells.sum() * grid.dx / grid.x_star)
    return rho_cells, g0, rho_bar
