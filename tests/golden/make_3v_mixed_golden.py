"""Golden vectors for the one-CTA-per-row big-row layout on partly kinetic
slices: the reference's default velocity grid (32 x 16 x 16, nx = 32), hybrid
runs whose labels stay mixed (38 % and 94 % kinetic) or shrink step by step to
all-fluid, so the device runs its sparse (listed-row) phases and the
kinetic -> fluid zeroing.  Straight from the REAL reference.

    python tests/golden/make_3v_mixed_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")

from make_3v_golden import digest, initial  # noqa: E402
from parakin.adaptation import Thresholds  # noqa: E402
from parakin.hybrid import HybridOptions, HybridState, hybrid_propagate  # noqa: E402
from parakin.kinetic import KineticStepParams  # noqa: E402
from parakin.lifting import lift  # noqa: E402
from parakin.mesh import MacroState, MeshSpec, MicroState, build_mesh  # noqa: E402
from parakin.poisson import solve_field  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
# (eps, threshold for both indicators): kinetic fraction over the 13 steps
CASES = [(1e-2, 1e-2), (1e-2, 1e-3), (1e-3, 1e-3)]


def main():
    out = {}
    m = build_mesh(MeshSpec(nx=32, nvx=32, nvy=16, nvz=16))
    rho, g0, rb = initial(m)
    E0 = solve_field(rho, rb, m)
    for eps, thr in CASES:
        k = f"{eps:g}_{thr:g}"
        p = KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
        gs = lift(rho, E0, eps, m, order=2, rho_bar=rb).g
        st = HybridState.initial(MacroState(rho, E0, 0.0), MicroState(gs), m)
        fr = []
        res = hybrid_propagate(st, 12.5 * p.dt, p, Thresholds(thr, thr), HybridOptions(), m, rb,
                               field_rtol=1.0,
                               trace=lambda s: fr.append(float(s.labels.kinetic_cells.mean())))
        out[k + "_dt"] = np.array(p.dt)
        out[k + "_frac"] = np.array(fr)
        out[k + "_rho"], out[k + "_E"], out[k + "_Ep"] = res.macro.rho, res.macro.E, res.E_prev
        out[k + "_kc"], out[k + "_ki"] = res.labels.kinetic_cells, res.labels.kinetic_ifaces
        out[k + "_g"] = np.array(digest(res.micro.g))
        print(k, "kinetic fraction per step", np.round(fr, 2))
    np.savez_compressed(os.path.join(OUT, "v3_mixed.npz"), **out)


if __name__ == "__main__":
    main()
