"""Golden artifact files written by the REAL reference's own writers.

Run in the build container (where /root/reference exists):

    python tests/golden/make_artifacts_golden.py

For three small 1V runs (two parareal PAR_CASES and one serial run with
parareal_enabled=False) it calls parakin's ``parareal.run`` and then the
writer functions of parakin/experiment.py:222-265 (boundaries, snapshots,
convergence, mass, labels) and writes the files to
tests/golden/artifacts/<case>/.  timings.csv is wall-clock dependent; its key
column is stored instead.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as MG  # noqa: E402  (imports parakin from /root/reference)

import parakin.experiment as ex  # noqa: E402
from parakin import parareal as ppl  # noqa: E402
from parakin.poisson import solve_field  # noqa: E402

OUT = Path(HERE) / "artifacts"
SNAPSHOTS = 3

# case -> (nx, nv, eps, adaptation, ng, T, k_max, tol, delta0, eta0, parareal_enabled);
# the two parareal cases are PAR_CASES "on_1e-4" and "off_0.5" (make_golden.py)
CASES = {
    "par_on_1e-4": (32, 16, 1e-4, True, 6, 0.3, 12, 1e-10, 1e-5, 1e-5, True),
    "par_off_0.5": (32, 16, 0.5, False, 6, 0.3, 12, 1e-10, 1e-5, 1e-5, True),
    "serial_off_0.5": (32, 16, 0.5, False, 6, 0.3, 12, 1e-10, 1e-5, 1e-5, False),
    "serial_on_0.5": (32, 16, 0.5, True, 6, 0.3, 12, 1e-10, 1e-5, 1e-5, False),
}


def main():
    for case, (nx, nv, eps, adapt, ng, T, kmax, tol, d0, e0, para) in CASES.items():
        m = MG.mesh1v(nx, nv)
        rho, g0, rb = MG.decompose(m, MG.f_paper(m))
        cfg = ppl.PararealConfig(eps=eps, t_final=T, ng=ng, k_max=kmax, tol=tol, workers=1,
                                 parareal_enabled=para, thresholds=MG.Thresholds(d0, e0),
                                 options=MG.HybridOptions(adaptation=adapt))
        res = ppl.run(cfg, rho, MG.g2(g0).reshape(g0.shape), m, rb)
        bounds = res.ledger.boundaries
        rtol = ppl.ADAPTIVE_FIELD_RTOL if adapt else None
        E = np.stack([solve_field(r, rb, m, rtol=rtol) for r in res.boundary_rho])
        ns = SimpleNamespace(eps=eps, t_final=T, snapshots=SNAPSHOTS, snapshot_times=(),
                             windows=ng, workers=1)
        out = OUT / case
        out.mkdir(parents=True, exist_ok=True)
        ex._write_boundaries(out, ns, m, bounds, res.boundary_rho, E)
        ex._write_snapshots(out, ns, m, bounds, res.boundary_rho, E)
        ex._write_convergence(out, ns, res)
        ex._write_mass(out, ns, m, bounds, res.boundary_rho)
        ex._write_labels(out, bounds, res.kinetic_fraction)
        ex._write_timings(out, ns, res, res.status, res.iterations, 0.0)
        keys = [line.split(",")[0] for line in (out / "timings.csv").read_text().splitlines()]
        (out / "timings.csv").unlink()
        (out / "timings_keys.txt").write_text("\n".join(keys) + "\n")
        print(case, res.status, res.iterations)


if __name__ == "__main__":
    main()
