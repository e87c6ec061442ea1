"""BASELINE cfg4 at its full grid, one parareal iteration at a reduced T, from
the oracle (the reference has no eps(x); the oracle restatement is
pinned bit for bit to the reference at constant eps).

cfg4 = Nx=8192, Nv=256, v*=10, eps(x) = 1e-3 + 0.5 exp(-20 (x - pi)^2),
delta0 = eta0 = 1e-3, 64 slices, seeded rho_in (configs.cfg4, seed 0).  The
full T = 2 needs 452,550 fine steps per window (CPU-infeasible), so T is
reduced to 64 x 100 fine steps at the reference dt: every window runs 100
hybrid steps, the coarse propagator 27 steps per window.  Recorded under the
reference's guard (it does not trip in this sample): the coarse sweep, all 64
windows' F, the kinetic fractions, the corrected row and err of iteration 1
(k_max = 1: status max_iterations), i.e. what ``run`` returns.

    python tests/golden/make_cfg4_golden.py [--procs N]     (~3 min on 8 cores)

Writes tests/golden/cfg4_iter1.npz.
"""

from __future__ import annotations

import os
import sys
import time
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

FINE_STEPS = 100


def setup():
    from oracle import restate as R
    from paper_2511_13386_b200 import configs

    c = configs.cfg4()
    g = R.make_grid(8192, 256, v_star=10.0)
    eps = R.EpsProfile.from_function(configs.eps_bump, g)
    rho0 = c.rho
    g0 = c.g.reshape(8192, 256)
    rb = c.rho_bar
    full = R.PConfig(eps=eps, t_final=2.0, ng=64, k_max=1, tol=1e-8, delta0=1e-3, eta0=1e-3,
                     opts=R.HOpts(adaptation=True))
    E0 = R.field(rho0, rb, g)
    dt_c, dt_f = R.default_steps(full, g, E0)
    cfg = R.PConfig(eps=eps, t_final=64 * FINE_STEPS * dt_f, ng=64, k_max=1, tol=1e-8,
                    delta0=1e-3, eta0=1e-3, opts=R.HOpts(adaptation=True))
    return R, g, eps, rho0, g0, rb, cfg, dt_c, dt_f


def _window(args):
    n, rho_in = args
    os.environ["OMP_NUM_THREADS"] = "1"
    R, g, eps, rho0, g0, rb, cfg, dt_c, dt_f = setup()
    F, frac = R.fine_window(n, rho_in, g0, cfg, dt_f, g, rb)
    return n, F, frac, F - R.coarse(rho_in, n, cfg, dt_c, g, rb)


def main():
    procs = int(sys.argv[sys.argv.index("--procs") + 1]) if "--procs" in sys.argv else os.cpu_count()
    tic = time.perf_counter()
    R, g, eps, rho0, g0, rb, cfg, dt_c, dt_f = setup()
    ng = cfg.ng
    row0 = np.empty((ng + 1, g.nx))
    row0[0] = rho0
    rho, t = rho0, 0.0
    for n in range(1, ng + 1):
        rho, _ = R.fluid_advance(rho, t, float(cfg.bounds[n]), dt_c, g, rb, None)
        t = float(cfg.bounds[n])
        row0[n] = rho
    with Pool(procs) as pool:
        res = sorted(pool.map(_window, [(n, row0[n - 1]) for n in range(ng, 0, -1)], chunksize=1),
                     key=lambda r: r[0])
    F = np.stack([r[1] for r in res])
    frac = np.array([r[2] for r in res])
    delta = np.stack([r[3] for r in res])
    new = row0.copy()
    for n in range(1, ng + 1):
        new[n] = R.coarse(new[n - 1], n, cfg, dt_c, g, rb) + delta[n - 1]
    err = float(np.max(np.abs(new - row0)))
    np.savez_compressed(os.path.join(HERE, "cfg4_iter1.npz"), row0=row0, frac=frac,
                        row1=new, err=np.array(err), dt_c=np.array(dt_c), dt_f=np.array(dt_f),
                        fine_steps=np.array(FINE_STEPS), t_final=np.array(cfg.t_final))
    print(f"cfg4 reduced-T iteration 1 via the oracle: {time.perf_counter() - tic:.0f} s, "
          f"err {err:.3e}, kinetic fractions {frac.min():.3f}..{frac.max():.3f}")


if __name__ == "__main__":
    main()
