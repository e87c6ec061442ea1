"""The reference's engine-level contracts (pkg/tests/test_parareal.py) re-run on
the drop-in's device engine, against values from the real reference
(tests/golden/make_golden.py, make_contract_golden.py):

* `max_iterations` is a status, not an error (parareal.py:333-353);
* prefix exactness (test_parareal.py:72-82): after k iterations rows n <= k
  equal the lift-restart chain -- through the drop-in's OWN
  ``lift_restart_reference`` (parareal.py:395-413), itself bitwise the
  reference's chain;
* worker-count independence (test_parareal.py:93-101): ``workers`` /
  PARAKIN_WORKERS never change the ledger;
* NonFiniteState (test_parareal.py:123-132): through the reference's seam
  (a blown-up ``_fine_window``) AND through the device path -- a non-finite
  window caught by the jump kernel, a non-finite row by the maxdiff kernel,
  in both schedules."""

import numpy as np
import pytest

import oracle as O
from _cases import f_paper

pytestmark = pytest.mark.gpu

pk = pytest.importorskip("paper_2511_13386_b200")
import paper_2511_13386_b200.parareal as ppl  # noqa: E402


def _paper(nx=32, nv=16):
    m = pk.build_mesh(pk.MeshSpec(nx=nx, nvx=nv))
    grid = O.make_grid(nx, nv)
    rho, g0, rb = O.decompose(f_paper(grid.vx, grid.M, grid.x_star), grid)
    return m, rho, g0.reshape(nx, nv, 1, 1), rb


def _cfg(k_max=12, workers=1, ng=6):
    return pk.PararealConfig(eps=0.5, t_final=0.3, ng=ng, k_max=k_max, tol=1e-10,
                             workers=workers, thresholds=pk.Thresholds(1e-5, 1e-5),
                             options=pk.HybridOptions(adaptation=False))


@pytest.mark.parametrize("overlap", [True, False])
def test_max_iterations_is_a_status(gold, monkeypatch, overlap):
    monkeypatch.setattr(ppl, "OVERLAP", overlap)
    d = gold("contracts")
    m, rho, g0, rb = _paper()
    res = pk.run(_cfg(k_max=3), rho, g0, m, rb)
    assert res.status == "max_iterations" and res.iterations == int(d["kmax_meta"][0])
    assert np.array_equal(np.stack(res.ledger.rho), d["kmax_rows"])
    assert np.array_equal(res.ledger.err, d["kmax_err"])


def test_prefix_exactness_through_dropin_chain(gold):
    d = gold("parareal")
    m, rho, g0, rb = _paper()
    cfg = _cfg()
    chain = ppl.lift_restart_reference(cfg, rho, g0, m, rb)
    assert np.array_equal(chain, d["p_off_0.5_chain"])      # the reference's own chain
    res = pk.run(cfg, rho, g0, m, rb)
    scale = np.max(np.abs(chain))
    for k, row in enumerate(res.ledger.rho):
        n = min(k, cfg.ng)
        assert np.max(np.abs(row[:n + 1] - chain[:n + 1])) <= 1e-12 * scale
        assert np.array_equal(row[0], rho)                   # initial row fixed


def test_worker_count_independence(gold, monkeypatch):
    d = gold("contracts")
    m, rho, g0, rb = _paper()
    rows = []
    for w in (1, 4):
        rows.append(np.stack(pk.run(_cfg(workers=w), rho, g0, m, rb).ledger.rho))
    monkeypatch.setenv(ppl.WORKERS_ENV, "8")
    rows.append(np.stack(pk.run(_cfg(), rho, g0, m, rb).ledger.rho))
    for r in rows:
        assert np.array_equal(r, d["w4_rows"])


def test_nonfinite_through_the_seam(monkeypatch):
    def blowup(n, rho_in, g0, cfg, kin_p, mesh, rho_bar, ws=None):
        return np.full_like(rho_in, np.inf), {"lift_s": 0.0, "fine_s": 0.0,
                                              "kinetic_fraction": 1.0}

    monkeypatch.setattr(ppl, "_fine_window", blowup)
    m, rho, g0, rb = _paper()
    with pytest.raises(pk.NonFiniteState):
        pk.run(_cfg(ng=3), rho, g0, m, rb)


@pytest.mark.parametrize("overlap", [True, False])
def test_nonfinite_through_device_kernels(monkeypatch, overlap):
    """A NaN boundary density: the field guard lets a NaN defect through (as
    Python's comparison does), F goes non-finite, and the device jump kernel
    flags it -- NonFiniteState for that window, in either schedule."""
    monkeypatch.setattr(ppl, "OVERLAP", overlap)
    m, rho, g0, rb = _paper()
    cfg = _cfg(ng=4)
    E0 = pk.solve_field(rho, rb, m)
    fluid_p, kin_p = ppl.default_params(cfg, m, E0)
    eng = ppl._Engine(cfg, m, rho, g0, rb, fluid_p, kin_p)
    eng.coarse_sweep()
    eng.row[2, 5] = float("nan")                 # the input of window 3
    with pytest.raises(pk.NonFiniteState, match="window 3"):
        eng.iterate(0)
    eng.close()
    # the maxdiff kernel on a non-finite new row (parareal.py:283-284)
    bad = eng.row.clone()
    bad[1, 0] = float("inf")
    with pytest.raises(pk.NonFiniteState):
        eng.be.maxdiff(bad, eng.row)
