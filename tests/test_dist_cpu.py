"""Multi-rank parareal coordination on CPU: world_size 2 over gloo.

The engine deals the active windows cyclically to ranks, all-gathers the fine
results and runs the correction on every rank.  Here the kernels are replaced
by the oracle backend, so this checks the coordination logic itself: both
ranks must hold identical ledgers, equal bit for bit to the single-process
reference run (tests/golden) — the multi-GPU analogue of the reference's
worker-count independence test (tests/test_parareal.py:93-101)."""

import os
import socket
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    for p in (ROOT, HERE):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        import paper_2511_13386_b200 as pk
        import paper_2511_13386_b200.parareal as ppl
        from _cases import f_paper
        from _oracle_backend import OracleBackend, oracle_solve_field

        name, nx, nv, eps, adapt, ng, T, kmax, tol, d0, e0 = case
        ppl._BACKEND = OracleBackend
        grid = O.make_grid(nx, nv)
        ppl.solve_field = oracle_solve_field(lambda m: grid)
        mesh = pk.build_mesh(pk.MeshSpec(nx=nx, nvx=nv))
        rho, g0, rb = O.decompose(f_paper(grid.vx, grid.M, grid.x_star), grid)
        cfg = pk.PararealConfig(eps=eps, t_final=T, ng=ng, k_max=kmax, tol=tol,
                                thresholds=pk.Thresholds(d0, e0),
                                options=pk.HybridOptions(adaptation=adapt))
        try:
            res = pk.run(cfg, rho, g0.reshape(nx, nv, 1, 1), mesh, rb)
        except pk.SimulationError as ex:
            np.savez(os.path.join(out_dir, f"r{world}_{rank}.npz"),
                     raised=np.array(type(ex).__name__), msg=np.array(str(ex)))
            return
        np.savez(os.path.join(out_dir, f"r{world}_{rank}.npz"), rows=np.stack(res.ledger.rho),
                 err=np.array(res.ledger.err), frac=res.kinetic_fraction,
                 meta=np.array([res.iterations, res.status == "converged"]))
    finally:
        dist.destroy_process_group()


CASES = [
    ("off_0.5", 32, 16, 0.5, False, 6, 0.3, 12, 1e-10, 1e-5, 1e-5),
    ("on_1e-4", 32, 16, 1e-4, True, 6, 0.3, 12, 1e-10, 1e-5, 1e-5),
]
# the reference raises SolvabilityViolation in this run (tests/golden: p_on_1e-2_raised)
RAISING = ("on_1e-2", 32, 16, 1e-2, True, 5, 0.2, 8, 1e-10, 1e-3, 1e-3)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_parareal_ranks_gloo(tmp_path, gold, case, world):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    d = gold("parareal")
    k = "p_" + case[0]
    for r in range(world):
        got = np.load(tmp_path / f"r{world}_{r}.npz")
        assert np.array_equal(got["rows"], d[k + "_rows"]), f"rank {r} ledger differs"
        assert np.array_equal(got["err"], d[k + "_err"])
        assert np.array_equal(got["frac"], d[k + "_frac"])
        assert list(got["meta"]) == list(d[k + "_meta"])


def test_parareal_ranks_failure_consensus(tmp_path, gold):
    """A fine window that trips the field guard on ONE rank must not leave the
    other ranks blocked in the all-gather: every rank raises the same error,
    that of the lowest failing window (the reference consumes its window
    futures in order, parareal.py:260-266), identical for 1, 2 and 3 ranks."""
    import torch.multiprocessing as mp

    assert bool(gold("parareal")["p_on_1e-2_raised"])
    msgs = set()
    for world in (1, 2, 3):
        mp.spawn(_worker, args=(world, _free_port(), RAISING, str(tmp_path)), nprocs=world,
                 join=True)
        got = [np.load(tmp_path / f"r{world}_{r}.npz") for r in range(world)]
        assert {str(g["raised"]) for g in got} == {"SolvabilityViolation"}
        msgs |= {str(g["msg"]) for g in got}
    assert len(msgs) == 1 and "window" in next(iter(msgs)), msgs
