"""Golden vectors for the reference-side seam binding (paper_2511_13386_b200.seam),
straight from the REAL reference's plugin seam ``parakin.parareal._fine_window``
(parareal.py:153-190) on its own default 1D-3V grid (nx=32, 32 x 16 x 16).

    python tests/golden/make_seam_golden.py

Windows 1 (true g0) and 2 (lifted restart) of two 4-window adaptive
configurations, both partly kinetic (eps 0.05 with OR labels, thresholds
0.03; eps 1e-3 with AND labels, thresholds 1; the adaptive field guard relaxed to 1.0 through the
reference's module attribute, as the seam reads it), plus the reference mesh / config values a duck-typed stand-in needs on a
box without the reference.  Writes tests/golden/seam.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import parakin.parareal as ppl  # noqa: E402
from parakin.adaptation import Thresholds  # noqa: E402
from parakin.hybrid import HybridOptions  # noqa: E402
from parakin.kinetic import KineticStepParams  # noqa: E402
from parakin.mesh import MeshSpec, build_mesh  # noqa: E402
from parakin.poisson import solve_field  # noqa: E402

from make_3v_golden import digest, initial  # noqa: E402


def main():
    m = build_mesh(MeshSpec(nx=32, nvx=32, nvy=16, nvz=16))
    rho, g0, rb = initial(m)
    E0 = solve_field(rho, rb, m)
    ppl.ADAPTIVE_FIELD_RTOL = 1.0
    out = {"spec": np.array([32, 32, 16, 16, m.x_star, m.v_star]),
           "vgrid": np.array([m.dx, m.vgrid.dv3, m.vgrid.m0, m.vgrid.m2]),
           "M": m.vgrid.M.reshape(-1), "vx": m.vgrid.vx, "rho0": rho, "rho_bar": np.array(rb),
           "g0_digest": np.array(digest(g0))}
    for case, eps, th, opts in (("or", 0.05, 0.03, HybridOptions()),
                                ("and", 1e-3, 1.0, HybridOptions(combine="and"))):
        p = KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
        cfg = ppl.PararealConfig(eps=eps, t_final=4 * 20.5 * p.dt, ng=4, k_max=3, tol=1e-10,
                                 workers=1, thresholds=Thresholds(th, th), options=opts)
        out[f"{case}_dt"] = np.array(p.dt)
        out[f"{case}_par"] = np.array([eps, th])
        out[f"{case}_t_final"] = np.array(cfg.t_final)
        rho_in = rho
        for n in (1, 2):
            r, diag = ppl._fine_window(n, rho_in, g0, cfg, p, m, rb)
            out[f"{case}_w{n}_in"] = rho_in
            out[f"{case}_w{n}_rho"] = r
            out[f"{case}_w{n}_frac"] = np.array(diag["kinetic_fraction"])
            print(case, "window", n, "kinetic fraction", diag["kinetic_fraction"])
            rho_in = r
    np.savez_compressed(os.path.join(HERE, "seam.npz"), **out)


if __name__ == "__main__":
    main()
