"""Golden vectors for 1D-3V grids (nvy, nvz >= 4: the reference's own mesh
family, mesh.py:58-65), straight from the REAL reference.

    python tests/golden/make_3v_golden.py

The reference runs through its public functions on its own 3V meshes; the
initial data is the paper recipe f0 = M(v) xi^4 (1 + 0.9 cos(2 pi x / x*))
decomposed as experiment.py:64-85 does.  Large arrays are stored as sha256
digests of their bytes.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from parakin.adaptation import Thresholds  # noqa: E402
from parakin.hybrid import HybridOptions, HybridState, hybrid_propagate  # noqa: E402
from parakin.kinetic import KineticStepParams, kinetic_propagate  # noqa: E402
from parakin.lifting import lift  # noqa: E402
from parakin.mesh import MacroState, MeshSpec, MicroState, build_mesh  # noqa: E402
from parakin.parareal import PararealConfig, run  # noqa: E402
from parakin.poisson import solve_field  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (nx, nvx, nvy, nvz): rows of one warp's registers (<= 256 nodes: even / odd
# nvx, a non-power-of-two nvy*nvz, the 256-node limit) and big rows (the
# reference's own test/default grid 32x32x16x16, odd nvx with a multi-leaf fold,
# a folded length whose pairwise split is not a power of two)
MESHES = [(16, 8, 4, 4), (12, 7, 4, 4), (10, 6, 5, 4), (16, 16, 4, 4),
          (32, 32, 16, 16), (16, 17, 8, 8), (12, 30, 8, 4)]


def digest(a) -> str:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return hashlib.sha256(a.tobytes()).hexdigest()


def initial(m):
    """experiment.py:64-85 for f0 = M xi^4 (1 + 0.9 cos(2 pi x / x*))."""
    grid = m.vgrid
    w = grid.xi**4 * grid.M

    def f(x):
        return w[None] * (1.0 + 0.9 * np.cos(2.0 * np.pi * x / m.x_star))[:, None, None, None]

    rho = m.bracket_x(f(m.x_centers))
    f_if = f(m.x_interfaces)
    g0 = f_if - m.bracket_x(f_if)[:, None, None, None] * grid.M[None]
    rb = float(rho.sum() * m.dx / m.x_star)
    return rho, g0, rb


def main():
    out = {}
    for nx, nvx, nvy, nvz in MESHES:
        k = f"{nx}_{nvx}_{nvy}_{nvz}"
        m = build_mesh(MeshSpec(nx=nx, nvx=nvx, nvy=nvy, nvz=nvz))
        g = m.vgrid
        out["M_" + k] = g.M.reshape(-1)
        out["s_" + k] = np.array([m.dx, g.dvx, g.dv3, g.m0, g.m2])
        rho, g0, rb = initial(m)
        out["in_" + k] = np.concatenate([rho, [rb]])
        out["g0_" + k] = np.array(digest(g0))
        E0 = solve_field(rho, rb, m)
        for eps in (0.5, 1e-4):
            p = KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
            mac, mic = kinetic_propagate((MacroState(rho, E0, 0.0), MicroState(g0)), 12.5 * p.dt,
                                         p, m, rb)
            kk = f"k_{k}_{eps:g}"
            out[kk + "_dt"] = np.array(p.dt)
            out[kk + "_rho"], out[kk + "_E"] = mac.rho, mac.E
            out[kk + "_g"] = np.array(digest(mic.g))
        # lift (order 2, both time eliminations)
        for te in ("leading", "higher_order"):
            dE = (E0 - 0.5 * E0) / 1e-3
            gl = lift(rho, E0, 1e-2, m, order=2, dE_dt=dE, time_elim=te, rho_bar=rb)
            out[f"l_{k}_{te}"] = np.array(digest(gl.g))
        # hybrid with adaptation: (a) from a lifted g, AND labels, lift re-init;
        # (b) the paper data, OR labels (make_golden.py's l_1e-3_and / p_0.5_or)
        for name, eps, start_lift, th, opts in (
                ("and", 1e-3, True, Thresholds(1e-2, 1e-2), HybridOptions(combine="and")),
                ("or", 0.5, False, Thresholds(1e-2, 1e-2), HybridOptions())):
            p = KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
            gs = lift(rho, E0, eps, m, order=2, rho_bar=rb).g if start_lift else g0
            st = HybridState.initial(MacroState(rho, E0, 0.0), MicroState(gs), m)
            res = hybrid_propagate(st, 40.5 * p.dt, p, th, opts, m, rb, field_rtol=1.0)
            hk = f"h_{k}_{name}"
            out[hk + "_dt"] = np.array(p.dt)
            out[hk + "_rho"], out[hk + "_E"], out[hk + "_Ep"] = res.macro.rho, res.macro.E, res.E_prev
            out[hk + "_kc"], out[hk + "_ki"] = res.labels.kinetic_cells, res.labels.kinetic_ifaces
            out[hk + "_g"] = np.array(digest(res.micro.g))
            print(k, name, "hybrid kinetic fraction", res.labels.kinetic_cells.mean())
    # a small parareal run on the first mesh
    m = build_mesh(MeshSpec(nx=16, nvx=8, nvy=4, nvz=4))
    rho, g0, rb = initial(m)
    cfg = PararealConfig(eps=0.5, t_final=0.2, ng=4, k_max=6, tol=1e-10, workers=1,
                         options=HybridOptions(adaptation=False))
    res = run(cfg, rho, g0, m, rb)
    out["p_rows"] = np.stack(res.ledger.rho)
    out["p_err"] = np.array(res.ledger.err)
    out["p_meta"] = np.array([res.iterations, res.status == "converged"])
    print("parareal", res.status, res.iterations)
    np.savez_compressed(os.path.join(OUT, "v3.npz"), **out)


if __name__ == "__main__":
    main()
