"""Phase-space mesh, host side (the reference's mesh.py:1-236 API).

The mesh is built on the host with numpy exactly as the reference builds it
(mirrored velocity centres, Maxwellian renormalised twice by the folded
bracket), and its velocity constants are uploaded verbatim to the device by
:mod:`paper_2511_13386_b200.engine`.  Two grid families: the reference's
1D-3V tensor grids (``nvy, nvz >= 4``, mesh.py:58-65) and the 1D-x/1D-v
reduction ``nvy == nvz == 1`` (exact, same arrays and arithmetic
with trivial vy/vz axes).  Arrays keep the reference's shapes: ``g`` is
``(nx, nvx, nvy, nvz)``; the device row of an interface is its
``nv = nvx * nvy * nvz`` values in that (C) order.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import MeshTooSmall

TWO_PI = 2.0 * np.pi


def gaussian_weight(v_sq):
    """exp(-|v|^2/2) / (2 pi)^(3/2) (mesh.py:31-33)."""
    return np.exp(-0.5 * v_sq) / TWO_PI**1.5


def _centers(n: int, v_star: float) -> np.ndarray:
    """Mirror-symmetric cell centres on [-v*, v*] (mesh.py:36-44)."""
    step = 2.0 * v_star / n
    pos = (np.arange(n // 2) + 0.5) * step
    if n % 2 == 0:
        return np.concatenate([-pos[::-1], pos])
    pos = (np.arange(n // 2) + 1.0) * step
    return np.concatenate([-pos[::-1], [0.0], pos])


@dataclass(frozen=True)
class MeshSpec:
    """Grid counts and domain sizes (mesh.py:47-65); ``nvy = nvz = 1`` selects
    the 1D-x/1D-v reduction."""

    nx: int
    nvx: int
    nvy: int = 1
    nvz: int = 1
    x_star: float = TWO_PI
    v_star: float = 8.0

    def validate(self) -> None:
        if self.nx < 7:
            raise MeshTooSmall(f"nx={self.nx}: spatial stencils need at least 7 cells")
        if self.nvx < 4:
            raise MeshTooSmall(f"nvx={self.nvx}: velocity grids need at least 4 cells")
        if (self.nvy, self.nvz) != (1, 1):
            for name, n in (("nvy", self.nvy), ("nvz", self.nvz)):
                if n < 4:
                    raise MeshTooSmall(f"{name}={n}: velocity grids need at least 4 cells")
        if self.x_star <= 0.0 or self.v_star <= 0.0:
            raise ValueError("x_star and v_star must be positive")


def _fold_sum(q: np.ndarray) -> np.ndarray:
    """<.> of (..., nvx, nvy, nvz) arrays without dv3 (mesh.py:95-133): fold the
    xi mirror pairs, numpy-sum the folded block over the three velocity axes
    (one pairwise sum over the flattened (nvx/2, nvy, nvz) block), plus the
    middle xi plane summed over (nvy, nvz) for odd nvx."""
    n = q.shape[-3]
    h = n // 2
    tot = (q[..., :h, :, :] + q[..., ::-1, :, :][..., :h, :, :]).sum(axis=(-3, -2, -1))
    if n % 2 == 1:
        tot = tot + q[..., h, :, :].sum(axis=(-2, -1))
    return tot


@dataclass(frozen=True)
class VelocityGrid:
    vx: np.ndarray
    vy: np.ndarray
    vz: np.ndarray
    dvx: float
    dv3: float
    M: np.ndarray          # (nvx, nvy, nvz)
    xi: np.ndarray         # (nvx, 1, 1)
    m0: float
    m2: float
    centers: np.ndarray = field(repr=False)

    @property
    def shape(self):
        return self.M.shape


def bracket(q: np.ndarray, grid: VelocityGrid) -> float:
    """<q> over the whole velocity grid (mesh.py:112-121)."""
    if q.shape != grid.shape:
        raise ValueError(f"expected shape {grid.shape}, got {q.shape}")
    return float(_fold_sum(q) * grid.dv3)


def bracket_staggered(q: np.ndarray, grid: VelocityGrid) -> np.ndarray:
    """Per-interface <q> of a (..., nvx, nvy, nvz) field (mesh.py:124-133)."""
    if q.shape[-3:] != grid.shape:
        raise ValueError(f"expected trailing shape {grid.shape}, got {q.shape}")
    return _fold_sum(q) * grid.dv3


@dataclass(frozen=True)
class MacroState:
    rho: np.ndarray
    E: np.ndarray
    t: float


@dataclass(frozen=True)
class MicroState:
    g: np.ndarray


class PhaseMesh:
    """Immutable discretisation (mesh.py:152-194)."""

    def __init__(self, spec: MeshSpec, vgrid: VelocityGrid):
        self.spec = spec
        self.vgrid = vgrid
        self.nx = spec.nx
        self.dx = spec.x_star / spec.nx
        self.x_star = spec.x_star
        self.v_star = spec.v_star
        self.x_centers = (np.arange(spec.nx) + 0.5) * self.dx
        self.x_interfaces = (np.arange(spec.nx) + 1.0) * self.dx
        self.xi_plus = np.maximum(vgrid.xi, 0.0)
        self.xi_minus = np.minimum(vgrid.xi, 0.0)
        self.xi_M = vgrid.xi * vgrid.M

    @property
    def nv(self) -> int:
        """Velocity nodes per interface row (nvx * nvy * nvz)."""
        return int(self.vgrid.M.size)

    @property
    def nvx(self) -> int:
        return self.vgrid.vx.shape[0]

    @property
    def nvyz(self) -> int:
        """Row stride of the xi axis (nvy * nvz; 1 for the 1D-x/1D-v reduction)."""
        return self.nv // self.nvx

    def bracket(self, q):
        return bracket(q, self.vgrid)

    def bracket_x(self, q):
        return bracket_staggered(q, self.vgrid)

    @staticmethod
    def roll_prev(a):
        return np.roll(a, 1, axis=0)

    @staticmethod
    def roll_next(a):
        return np.roll(a, -1, axis=0)

    def iface_to_center(self, q):
        return 0.5 * (self.roll_prev(q) + q)

    def center_to_iface(self, q):
        return 0.5 * (q + self.roll_next(q))

    def g_shape(self):
        return (self.nx,) + self.vgrid.shape


def build_mesh(spec: MeshSpec) -> PhaseMesh:
    """mesh.py:197-236 (deterministic; identical specs give identical grids)."""
    spec.validate()
    vx = _centers(spec.nvx, spec.v_star)
    vy = _centers(spec.nvy, spec.v_star)
    vz = _centers(spec.nvz, spec.v_star)
    dvx = 2.0 * spec.v_star / spec.nvx
    dv3 = dvx * (2.0 * spec.v_star / spec.nvy) * (2.0 * spec.v_star / spec.nvz)
    v_sq = vx[:, None, None] ** 2 + vy[None, :, None] ** 2 + vz[None, None, :] ** 2
    M = gaussian_weight(v_sq)
    xi = vx[:, None, None]
    centers = np.stack(np.broadcast_arrays(vx[:, None, None], vy[None, :, None],
                                           vz[None, None, :]), axis=-1)

    def grid(M_, m0=0.0, m2=0.0):
        return VelocityGrid(vx=vx, vy=vy, vz=vz, dvx=dvx, dv3=dv3, M=M_, xi=xi,
                            m0=m0, m2=m2, centers=centers)

    for _ in range(2):
        M = M / bracket(M, grid(M))
    g = grid(M)
    return PhaseMesh(spec, grid(M, m0=bracket(M, g), m2=bracket(xi**2 * M, g)))
