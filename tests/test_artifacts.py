"""Run artifacts (paper_2511_13386_b200/artifacts.py) against files written
by the reference's own writers (tests/golden/make_artifacts_golden.py):
byte-identical boundaries/snapshots/convergence/mass/labels.csv, same
timings.csv keys."""

import os

import numpy as np
import pytest

import oracle as O
from _cases import f_paper

from paper_2511_13386_b200 import artifacts as A
from paper_2511_13386_b200.adaptation import Thresholds
from paper_2511_13386_b200.hybrid import HybridOptions
from paper_2511_13386_b200.parareal import (ADAPTIVE_FIELD_RTOL, PararealConfig, PararealLedger,
                                            RunResult)

GOLD = os.path.join(os.path.dirname(__file__), "golden", "artifacts")
FILES = ["boundaries.csv", "snapshots.csv", "convergence.csv", "mass.csv", "labels.csv"]
# case -> (nx, nv, eps, adaptation, ng, T, k_max, tol, delta0, eta0, parareal_enabled)
CASES = {
    "par_on_1e-4": (32, 16, 1e-4, True, 6, 0.3, 12, 1e-10, 1e-5, 1e-5, True),
    "par_off_0.5": (32, 16, 0.5, False, 6, 0.3, 12, 1e-10, 1e-5, 1e-5, True),
    "serial_off_0.5": (32, 16, 0.5, False, 6, 0.3, 12, 1e-10, 1e-5, 1e-5, False),
    "serial_on_0.5": (32, 16, 0.5, True, 6, 0.3, 12, 1e-10, 1e-5, 1e-5, False),
}


def config(case):
    nx, nv, eps, adapt, ng, T, kmax, tol, d0, e0, para = CASES[case]
    return PararealConfig(eps=eps, t_final=T, ng=ng, k_max=kmax, tol=tol, parareal_enabled=para,
                          thresholds=Thresholds(d0, e0), options=HybridOptions(adaptation=adapt))


def read(case, name):
    with open(os.path.join(GOLD, case, name), "rb") as fh:
        return fh.read()


def compare(case, paths):
    for name in FILES:
        with open(paths[name], "rb") as fh:
            assert fh.read() == read(case, name), f"{case}/{name} differs from the reference's"
    keys = [ln.split(",")[0] for ln in open(paths["timings.csv"]).read().splitlines()]
    assert keys == read(case, "timings_keys.txt").decode().split()


def snapshot_times(case):
    cfg = config(case)
    return A.default_snapshot_times(cfg.t_final, 3)


@pytest.mark.parametrize("case", list(CASES))
def test_writers_reproduce_reference_bytes(case, tmp_path):
    """CPU: rebuild each run's arrays from the reference's boundaries.csv (17
    significant digits round-trip doubles exactly), labels and errors, and
    write them again: every byte must match."""
    cfg = config(case)
    nx = CASES[case][0]
    rows = [ln.split(",") for ln in read(case, "boundaries.csv").decode().splitlines()[1:]]
    rho = np.array([float(r[4]) for r in rows]).reshape(cfg.ng + 1, nx)
    E = np.array([float(r[5]) for r in rows]).reshape(cfg.ng + 1, nx)
    lab = [ln.split(",") for ln in read(case, "labels.csv").decode().splitlines()[1:]]
    err = [float(ln.split(",")[2]) for ln in read(case, "convergence.csv").decode().splitlines()[1:]]
    ledger = PararealLedger(boundaries=cfg.boundaries, rho=[rho], err=err)
    res = RunResult(status="converged" if cfg.parareal_enabled else "serial",
                    iterations=len(err), ledger=ledger, boundary_rho=rho,
                    kinetic_fraction=np.array([float(r[1]) for r in lab]), config=cfg)
    grid = O.make_grid(nx, CASES[case][1])
    rb = O.decompose(f_paper(grid.vx, grid.M, grid.x_star), grid)[2]
    rtol = ADAPTIVE_FIELD_RTOL if cfg.options.adaptation else None
    E_oracle = np.stack([O.field(r, rb, grid, rtol) for r in rho])
    assert np.array_equal(E_oracle, E)  # the oracle's field of the reference's rows
    paths = A.write_run_artifacts(tmp_path, res, grid, 0.0, snapshot_times=snapshot_times(case),
                                  boundary_E=E, wall_s=0.0)
    for name in ["boundaries.csv", "snapshots.csv", "mass.csv", "labels.csv", "convergence.csv"]:
        with open(paths[name], "rb") as fh:
            assert fh.read() == read(case, name)


@pytest.mark.gpu
@pytest.mark.parametrize("case", list(CASES))
def test_run_artifacts_match_reference(case, tmp_path):
    """GPU: the drop-in run() (parareal or serial) and the writers reproduce
    the reference's artifact files byte for byte."""
    import paper_2511_13386_b200 as pk

    nx, nv = CASES[case][:2]
    m = pk.build_mesh(pk.MeshSpec(nx=nx, nvx=nv))
    grid = O.make_grid(nx, nv)
    rho, g0, rb = O.decompose(f_paper(grid.vx, grid.M, grid.x_star), grid)
    res = pk.run(config(case), rho, np.asarray(g0).reshape(m.nx, m.nv, 1, 1), m, rb)
    paths = A.write_run_artifacts(tmp_path, res, m, rb, snapshot_times=snapshot_times(case))
    compare(case, paths)
