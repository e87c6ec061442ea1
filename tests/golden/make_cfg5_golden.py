"""BASELINE cfg5 at the bench's full size, pinned to the REAL reference.

All 256 seeded instances of 1024x128 advanced 500 ``kinetic_step`` calls each
at ``KineticStepParams.default(mesh, eps_s, e_max=max|E0_s|)`` -- exactly the
work one ``bench.py`` step does -- through the reference's own public
functions (parakin.kinetic.kinetic_step, kinetic.py:255-273), one process per
core.  Stored: per instance sha256 digests of rho, E and g after 500 steps (NaNs
canonicalised), the step at which rho first turned non-finite (-1: never;
the reference's own stable dt is NOT stable for every instance: 7 of 256,
eps ~3.1e-4..3.3e-4 at the parabolic-bound dt, blow up -- the device must
reproduce that too),
the dt and rho_bar used, and the full rho/E arrays of four instances chosen
to sit at software-group / CTA boundaries of the bench launch (0, 3, 130,
255).

    python tests/golden/make_cfg5_golden.py [--procs N]

Runs in the build container (needs /root/reference); ~80 s on 8 cores.
Writes tests/golden/cfg5_500.npz.
"""

from __future__ import annotations

import os
import sys
import time
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

NSTEPS = 500
FULL = (0, 3, 130, 255)


def _job(s):
    os.environ["OMP_NUM_THREADS"] = "1"
    import make_golden as mg
    from parakin.kinetic import KineticStepParams, kinetic_step
    from parakin.mesh import MacroState, MicroState
    from parakin.poisson import solve_field

    m = mg.mesh1v(1024, 128)
    rho, g0, rb = mg.decompose(m, mg.f_cfg5(m, s))
    _, _, eps = mg.cfg5_instance(s)
    E0 = solve_field(rho, rb, m)
    p = KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
    st = (MacroState(rho, E0, 0.0), MicroState(g0))
    blowup = -1
    for i in range(NSTEPS):
        st = kinetic_step(st, p, m, rb)
        if blowup < 0 and not np.isfinite(st[0].rho).all():
            blowup = i
    mac, mic = st
    return (s, cdigest(mac.rho), cdigest(mac.E), cdigest(mg.g2(mic.g)), p.dt, rb,
            mac.rho if s in FULL else None, mac.E if s in FULL else None, blowup, eps)


def cdigest(a):
    """sha256 of the fp64 bytes with every NaN replaced by numpy's canonical
    quiet NaN (x86 and the GPU produce different NaN payloads/signs)."""
    a = np.array(a, dtype=np.float64, copy=True)
    a[np.isnan(a)] = np.nan
    import make_golden as mg

    return mg.digest(a)


def main():
    procs = int(sys.argv[sys.argv.index("--procs") + 1]) if "--procs" in sys.argv else os.cpu_count()
    tic = time.perf_counter()
    with Pool(procs) as pool:
        res = sorted(pool.map(_job, range(256), chunksize=1))
    out = {
        "rho_digest": np.array([r[1] for r in res]),
        "E_digest": np.array([r[2] for r in res]),
        "g_digest": np.array([r[3] for r in res]),
        "dt": np.array([r[4] for r in res]),
        "rho_bar": np.array([r[5] for r in res]),
        "blowup_step": np.array([r[8] for r in res]),
        "eps": np.array([r[9] for r in res]),
        "full_ids": np.array(FULL),
        "nsteps": np.array(NSTEPS),
    }
    for r in res:
        if r[0] in FULL:
            out[f"rho_{r[0]}"], out[f"E_{r[0]}"] = r[6], r[7]
    np.savez_compressed(os.path.join(HERE, "cfg5_500.npz"), **out)
    print(f"cfg5 x 256 x {NSTEPS} steps through the reference: {time.perf_counter() - tic:.1f} s "
          f"on {procs} processes")


if __name__ == "__main__":
    main()
