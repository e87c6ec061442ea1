"""Golden vectors for the reference's engine-level contracts re-run on the
drop-in (tests/test_contracts.py), from the REAL reference:

* `max_iterations` as a status, not an error (parareal.py:333-353): the
  32x16 paper-data case of make_golden.py's PAR_CASES "off_0.5" with
  k_max = 3 (it needs 7 iterations to converge);
* the worker-count contract's ledger at workers = 4 (parareal.py:17-20).

    python tests/golden/make_contract_golden.py     (writes contracts.npz)
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg  # noqa: E402  (imports the reference from /root/reference)
from parakin.adaptation import Thresholds  # noqa: E402
from parakin.hybrid import HybridOptions  # noqa: E402
from parakin.parareal import PararealConfig, run  # noqa: E402


def main():
    m = mg.mesh1v(32, 16)
    rho, g0, rb = mg.decompose(m, mg.f_paper(m))
    out = {}
    cfg = PararealConfig(eps=0.5, t_final=0.3, ng=6, k_max=3, tol=1e-10, workers=1,
                         thresholds=Thresholds(1e-5, 1e-5), options=HybridOptions(adaptation=False))
    res = run(cfg, rho, mg.g2(g0).reshape(g0.shape), m, rb)
    assert res.status == "max_iterations"
    out["kmax_rows"] = np.stack(res.ledger.rho)
    out["kmax_err"] = np.array(res.ledger.err)
    out["kmax_meta"] = np.array([res.iterations])
    cfg4 = PararealConfig(eps=0.5, t_final=0.3, ng=6, k_max=12, tol=1e-10, workers=4,
                          thresholds=Thresholds(1e-5, 1e-5), options=HybridOptions(adaptation=False))
    res4 = run(cfg4, rho, mg.g2(g0).reshape(g0.shape), m, rb)
    out["w4_rows"] = np.stack(res4.ledger.rho)
    np.savez_compressed(os.path.join(HERE, "contracts.npz"), **out)
    print("max_iterations after", res.iterations, "; workers=4 iterations", res4.iterations)


if __name__ == "__main__":
    main()
