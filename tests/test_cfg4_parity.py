"""BASELINE cfg4 at its full grid (8192 x 256, v* = 10, eps(x), 64 slices):
one parareal iteration at a reduced T (100 fine steps per window; the full
T = 2 needs 452,550) through the drop-in ``run()``, against the oracle
fixture tests/golden/make_cfg4_golden.py -- the coarse sweep, all 64
windows' F (the nv = 256 producer/consumer micro phase, the global-memory
slice phase run by every CTA of the cluster), the kinetic fractions, the
corrected row and err: bitwise in exact mode; masks identical and 1e-10
relative L2 in fast mode."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pk = pytest.importorskip("paper_2511_13386_b200")
from paper_2511_13386_b200 import configs  # noqa: E402
import paper_2511_13386_b200.parareal as ppl  # noqa: E402


def _run(d):
    c = configs.cfg4()
    m = c.mesh
    th = pk.Thresholds(1e-3, 1e-3)
    full = pk.PararealConfig(eps=c.eps, t_final=2.0, ng=64, k_max=1, tol=1e-8, thresholds=th,
                             options=pk.HybridOptions(adaptation=True))
    E0 = pk.solve_field(c.rho, c.rho_bar, m)
    fluid_p, kin_p = ppl.default_params(full, m, E0)
    assert kin_p.dt == float(d["dt_f"]) and fluid_p.dt == float(d["dt_c"])
    cfg = pk.PararealConfig(eps=c.eps, t_final=float(d["t_final"]), ng=64, k_max=1, tol=1e-8,
                            thresholds=th, options=pk.HybridOptions(adaptation=True))
    return pk.run(cfg, c.rho, c.g, m, c.rho_bar)


def test_cfg4_reduced_T_iteration1_bitwise(gold):
    d = gold("cfg4_iter1")
    res = _run(d)
    assert res.status == "max_iterations" and res.iterations == 1
    assert np.array_equal(res.ledger.rho[0], d["row0"])
    assert np.array_equal(res.ledger.rho[1], d["row1"])
    assert res.ledger.err[0] == float(d["err"])
    assert np.array_equal(res.kinetic_fraction[1:], d["frac"])
    assert 0.0 < d["frac"][1:].min() and d["frac"].max() < 1.0   # mixed kinetic / fluid


def test_cfg4_reduced_T_iteration1_fast_mode(gold):
    d = gold("cfg4_iter1")
    with pk.scan_mode(False):
        res = _run(d)
    assert res.status == "max_iterations"
    assert np.array_equal(res.kinetic_fraction[1:], d["frac"])
    for k, ref in ((0, d["row0"]), (1, d["row1"])):
        got = res.ledger.rho[k]
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-10
    assert abs(res.ledger.err[0] - float(d["err"])) <= 1e-6 * float(d["err"])
