"""Run artifacts in the reference's CSV formats (experiment.py:115-301).

Numbers are written with 17 significant digits (``%.17g``), headers and row
order as the reference writes them, so a run whose boundary rows, errors and
kinetic fractions equal the reference's bit for bit also produces its files
byte for byte (tests/test_artifacts.py against files written by the
reference's own writers, tests/golden/make_artifacts_golden.py).  Only
timings.csv depends on the wall clock.

The experiment front door (RunConfig, INI parsing, CLI) stays out of scope
(DESIGN.md §6): these writers take a ``RunResult`` from ``run()``.
"""

from __future__ import annotations

import csv
import os

import numpy as np

from .parareal import PerfModel, RunResult, predict_cost

FMT = "%.17g"


def fmt(x) -> str:
    return FMT % float(x)


def write_csv(path, header, rows) -> None:
    """experiment.py:115-119 (csv module, '\\n' line ends)."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(header)
        w.writerows(rows)


def default_snapshot_times(t_final: float, snapshots: int) -> np.ndarray:
    """config.py:207-214 without explicit times: one snapshot at t_final, else
    `snapshots` log-spaced times in [t_final/64, t_final]."""
    if snapshots == 1:
        return np.asarray([t_final])
    return np.geomspace(t_final / 64.0, t_final, snapshots)


def snapshot_rows(bounds, times) -> list[int]:
    """Boundary indices nearest the requested times (experiment.py:233-236)."""
    bounds = np.asarray(bounds, dtype=float)
    return sorted({int(np.argmin(np.abs(bounds - t))) for t in np.sort(np.asarray(times, float))})


def _eps_text(eps) -> str:
    try:
        return fmt(eps)
    except TypeError:  # an eps(x) profile (an extension; the reference's eps is a scalar)
        return "eps(x)"


def write_run_artifacts(out_dir, result: RunResult, mesh, rho_bar, *, snapshot_times=None,
                        wall_s: float | None = None, workers: int = 1, boundary_E=None) -> dict:
    """Write boundaries/snapshots/convergence/mass/labels/timings.csv for one run.

    ``boundary_E`` defaults to the field of every boundary row under the run's
    guard (``RunResult.boundary_fields``, experiment.py:160-163).  Returns the
    written paths by name."""
    os.makedirs(out_dir, exist_ok=True)
    cfg = result.config
    eps = _eps_text(cfg.eps)
    bounds = np.asarray(result.ledger.boundaries, dtype=float)
    rho = np.asarray(result.boundary_rho, dtype=float)
    E = result.boundary_fields(mesh, rho_bar) if boundary_E is None else np.asarray(boundary_E)
    x = mesh.x_centers
    paths = {}

    def out(name):
        paths[name] = os.path.join(out_dir, name)
        return paths[name]

    write_csv(out("boundaries.csv"), ["eps", "n", "t", "x", "rho", "E"],
              [(eps, str(n), fmt(t), fmt(x[i]), fmt(rho[n, i]), fmt(E[n, i]))
               for n, t in enumerate(bounds) for i in range(mesh.nx)])
    if snapshot_times is not None:
        write_csv(out("snapshots.csv"), ["t", "x", "rho", "E"],
                  [(fmt(bounds[n]), fmt(x[i]), fmt(rho[n, i]), fmt(E[n, i]))
                   for n in snapshot_rows(bounds, snapshot_times) for i in range(mesh.nx)])
    write_csv(out("convergence.csv"), ["eps", "k", "err"],
              [(eps, str(k), fmt(e)) for k, e in enumerate(result.ledger.err, start=1)])
    m0 = rho[0].sum() * mesh.dx
    write_csv(out("mass.csv"), ["eps", "n", "t", "dm"],
              [(eps, str(n), fmt(t), fmt(rho[n].sum() * mesh.dx - m0)) for n, t in enumerate(bounds)])
    write_csv(out("labels.csv"), ["t", "kinetic_fraction"],
              [(fmt(t), fmt(f)) for t, f in zip(bounds, result.kinetic_fraction)])
    tm = result.ledger.timings
    rows = [("status", result.status), ("iterations", str(result.iterations)),
            ("windows", str(cfg.ng)), ("workers", str(workers)), ("eps", eps),
            ("wall_total_s", fmt(tm.wall_total if wall_s is None else wall_s)),
            ("coarse_sweep_s", fmt(tm.coarse_sweep)), ("fine_window_max_s", fmt(tm.fine_max)),
            ("fine_total_s", fmt(tm.fine_total)), ("lift_window_max_s", fmt(tm.lift_max)),
            ("lift_total_s", fmt(tm.lift_total)),
            ("fluid_window_max_s", fmt(tm.fluid_window_max)),
            ("correction_total_s", fmt(tm.correction_total))]
    if result.iterations > 0:
        t_pred, k_opt, beats = predict_cost(PerfModel(
            t_hmm=tm.fine_max, t_fluid=tm.fluid_window_max, t_lift=tm.lift_max,
            n_workers=workers, ng=cfg.ng, k=result.iterations))
        rows += [("predicted_t_parareal_s", fmt(t_pred)), ("predicted_k_opt", str(k_opt)),
                 ("predicted_break_even", "yes" if beats else "no")]
    rows += [(f"iteration_{it['k']}_wall_s", fmt(it["wall_s"])) for it in tm.iterations]
    write_csv(out("timings.csv"), ["key", "value"], rows)
    return paths
