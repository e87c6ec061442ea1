"""The multi-rank parareal engine on the REAL device path: two ranks, each
running its share of the fine windows through libpk (DeviceBackend) on the
one GPU of the test box, exchanging results through the engine's all-gather
(gloo, staged through host memory).  The ranks' kernels are independent (no
rank waits on another's kernel), so sharing a GPU only serialises them.  The
ledger of BASELINE cfg2 must equal the reference's bit for bit on every rank
(cf. the reference's worker-count independence, tests/test_parareal.py:93-101)."""

import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, which, overlap=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    for p in (ROOT, HERE):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_13386_b200 as pk
        import paper_2511_13386_b200.parareal as ppl
        from paper_2511_13386_b200 import configs

        ppl.OVERLAP = overlap

        if which == "cfg2":
            c = configs.cfg2()
            cfg = pk.PararealConfig(eps=1e-2, t_final=0.5, ng=16, k_max=5, tol=1e-10,
                                    options=pk.HybridOptions(adaptation=False))
        else:   # cfg3 under the reference guard: raises on every rank, no hang
            c = configs.cfg3()
            cfg = pk.PararealConfig(eps=c.eps, t_final=1.0, ng=32, k_max=50, tol=1e-8,
                                    thresholds=pk.Thresholds(1e-3, 1e-3),
                                    options=pk.HybridOptions(adaptation=True))
        try:
            res = pk.run(cfg, c.rho, c.g, c.mesh, c.rho_bar)
        except pk.SimulationError as ex:
            np.savez(os.path.join(out_dir, f"{which}_{rank}.npz"),
                     raised=np.array(type(ex).__name__), msg=np.array(str(ex)))
            return
        np.savez(os.path.join(out_dir, f"{which}_{rank}.npz"), rows=np.stack(res.ledger.rho),
                 err=np.array(res.ledger.err), meta=np.array([res.iterations]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overlap", [True, False], ids=["overlapped", "phase-by-phase"])
def test_cfg2_two_ranks_device_engine(tmp_path, gold, overlap):
    """Overlapped: per-window payload broadcasts in window order feed every
    rank's own correction; phase-by-phase: one all-gather per iteration."""
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), "cfg2", overlap), nprocs=2,
             join=True)
    d = gold("parareal")
    for r in range(2):
        got = np.load(tmp_path / f"cfg2_{r}.npz")
        assert np.array_equal(got["rows"], d["c2_rows"]), f"rank {r} ledger differs"
        assert np.array_equal(got["err"], d["c2_err"])
        assert int(got["meta"][0]) == int(d["c2_meta"][0])


@pytest.mark.parametrize("overlap", [True, False], ids=["overlapped", "phase-by-phase"])
def test_cfg3_two_ranks_failure_consensus(tmp_path, gold, overlap):
    """Windows 2..32 all trip the reference guard (fixture); rank 1 holds
    window 2: both ranks must raise window 2's error at the oracle's step."""
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), "cfg3", overlap), nprocs=2,
             join=True)
    trips = gold("cfg3_iter1")["ref_trip"]
    first = min(n + 1 for n in range(32) if trips[n, 0] >= 0)
    for r in range(2):
        got = np.load(tmp_path / f"cfg3_{r}.npz")
        assert str(got["raised"]) == "SolvabilityViolation"
        assert f"window {first}, step {trips[first - 1, 0]}" in str(got["msg"])
