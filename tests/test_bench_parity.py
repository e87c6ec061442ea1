"""The bench workload itself, pinned: BASELINE cfg5 exactly as one
``bench.py`` step runs it (256 instances of 1024x128 in ONE launch of the
software-group layout, 500 steps at the reference stable dt) against the
reference's own results for every instance (tests/golden/make_cfg5_golden.py,
generated with /root/reference's parakin.kinetic.kinetic_step).  Bitwise,
NaNs canonicalised: 7 instances blow up under the reference's own dt."""

import os
import sys

import numpy as np
import pytest

from _cases import cdigest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cfg5_bench_launch_500_steps_vs_reference(gold):
    import torch

    sys.path.insert(0, ROOT)
    import bench
    from paper_2511_13386_b200.ensemble import Ensemble

    d = gold("cfg5_500")
    m, cases, rho0, g0, eps, rb, dts = bench.build_inputs(list(range(bench.NINST)))
    assert np.array_equal(np.array(dts), d["dt"]) and np.array_equal(np.array(rb), d["rho_bar"])
    ens = Ensemble(m, eps, dts, rb)
    ens.load(torch.from_numpy(rho0).cuda(), torch.from_numpy(g0).cuda())
    ens.run(int(d["nsteps"]))
    C, K, on_chip, kind = ens.dev.last_launch()
    if "PK_NO_SG" not in os.environ:
        assert kind == 1 and 1 < K < C, (C, K, kind)   # the bench's software-group layout
    rho, E, g = (x.cpu().numpy() for x in (ens.rho, ens.E, ens.g))
    bad = [s for s in range(bench.NINST)
           if (cdigest(rho[s]), cdigest(E[s]), cdigest(g[s]))
           != (d["rho_digest"][s], d["E_digest"][s], d["g_digest"][s])]
    assert not bad, f"instances differing from the reference: {bad}"
    for s in d["full_ids"]:
        assert np.array_equal(rho[s], d[f"rho_{s}"], equal_nan=True)
        assert np.array_equal(E[s], d[f"E_{s}"], equal_nan=True)
    blown = np.where(d["blowup_step"] >= 0)[0]
    assert len(blown) == 7 and all(not np.isfinite(rho[s]).all() for s in blown)
