"""BASELINE.json workloads: meshes, seeded initial data and step rules.

Initial data follow the reference's decomposition recipe
(experiment.py:64-85): rho = <f(x_i)>, g = f(x_{i+1/2}) - <f(x_{i+1/2})> M,
rho_bar = sum(rho) dx / x*.  The seeded conventions for cfg4/cfg5 are the
ones frozen in BASELINE.md §4.  Synthetic data stand in for the configs; no
dataset is involved.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .kinetic import EpsProfile
from .mesh import MeshSpec, PhaseMesh, build_mesh


@dataclass
class Case:
    mesh: PhaseMesh
    rho: np.ndarray        # (nx,)
    g: np.ndarray          # (nx, nv, 1, 1)
    rho_bar: float
    eps: object


def decompose(mesh: PhaseMesh, f_of_x):
    """experiment.py:64-85 for an arbitrary f(x) -> (len(x), nv)."""
    dv3 = mesh.vgrid.dv3
    M = mesh.vgrid.M.reshape(-1)

    def vs(q):
        n = q.shape[-1]
        h = n // 2
        t = (q[..., :h] + q[..., ::-1][..., :h]).sum(axis=-1)
        if n % 2:
            t = t + q[..., h]
        return t * dv3

    rho = vs(f_of_x(mesh.x_centers))
    f_if = f_of_x(mesh.x_interfaces)
    g = f_if - vs(f_if)[:, None] * M
    rho_bar = float(rho.sum() * mesh.dx / mesh.x_star)
    return rho, g.reshape((mesh.nx,) + mesh.vgrid.shape), rho_bar


def mesh1v(nx, nv, v_star=8.0):
    return build_mesh(MeshSpec(nx=nx, nvx=nv, v_star=v_star))


def cfg1(nx=128, nv=64):
    m = mesh1v(nx, nv)
    M = m.vgrid.M.reshape(-1)
    rho, g, rb = decompose(m, lambda x: (1.0 + 0.5 * np.cos(x))[:, None] * M[None, :])
    return Case(m, rho, g, rb, 1.0)


def cfg2(nx=256, nv=64, eps=1e-2):
    m = mesh1v(nx, nv)
    M = m.vgrid.M.reshape(-1)
    vM = m.vgrid.vx * M
    rho, g, rb = decompose(m, lambda x: ((1.0 + 0.3 * np.cos(x) + 0.1 * np.sin(2.0 * x))[:, None]
                                         * M[None, :]
                                         + (1e-3 * eps) * np.cos(x)[:, None] * vM[None, :]))
    return Case(m, rho, g, rb, eps)


def eps_bump(x):
    """cfg3/cfg4 eps(x) = 1e-3 + 0.5 exp(-20 (x - pi)^2)."""
    return 1e-3 + 0.5 * np.exp(-20.0 * (x - np.pi) ** 2)


def cfg3(nx=512, nv=128):
    m = mesh1v(nx, nv)
    M = m.vgrid.M.reshape(-1)
    rho, g, rb = decompose(m, lambda x: (1.0 + 0.5 * np.cos(x))[:, None] * M[None, :])
    return Case(m, rho, g, rb, EpsProfile.from_function(eps_bump, m))


def cfg4(nx=8192, nv=256, seed=0):
    m = mesh1v(nx, nv, v_star=10.0)
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.0, 0.05, 8)
    ph = rng.uniform(0.0, 2.0 * np.pi, 8)
    M = m.vgrid.M.reshape(-1)

    def f(x):
        r = np.ones_like(x)
        for k in range(8):
            r = r + a[k] * np.cos((k + 1) * x + ph[k])
        return r[:, None] * M[None, :]

    rho, g, rb = decompose(m, f)
    return Case(m, rho, g, rb, EpsProfile.from_function(eps_bump, m))


def cfg5_instance(s):
    rng = np.random.default_rng(s)
    a = rng.uniform(0.0, 0.1, 4)
    ph = rng.uniform(0.0, 2.0 * np.pi, 4)
    eps = float(10.0 ** rng.uniform(-4.0, 0.0))
    return a, ph, eps


def cfg5(instances=range(256), nx=1024, nv=128, mesh=None):
    """Ensemble: list of Case, one per seeded instance (shared mesh)."""
    m = mesh or mesh1v(nx, nv)
    M = m.vgrid.M.reshape(-1)
    vx = m.vgrid.vx
    out = []
    for s in instances:
        a, ph, eps = cfg5_instance(s)

        def f(x, a=a, ph=ph):
            r = np.ones_like(x)
            for k in range(4):
                r = r + a[k] * np.cos((k + 1) * x + ph[k])
            return (r[:, None] * M[None, :]) * (1.0 + 0.01 * vx[None, :] * np.cos(x)[:, None])

        rho, g, rb = decompose(m, f)
        out.append(Case(m, rho, g, rb, eps))
    return out
