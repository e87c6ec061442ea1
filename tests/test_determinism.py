"""Run-to-run bitwise determinism of every cross-CTA synchronisation protocol
under perturbed timing (compute-sanitizer is closed on this GPU pool -- see
DESIGN.md §6 -- so races are hunted this way): the software-group layout
(signalling-NaN sentinel moments + counter barrier), packed and single
clusters (DSMEM moments, cluster barriers), the hybrid slice phase in global
memory run by every CTA of a cluster (DSMEM list counters, cluster scans),
and the one-CTA-per-row big 1D-3V rows (TMA half-row staging).  Each case is
repeated with a memory-bound torch kernel running concurrently on another
stream (so CTAs reach the barriers in different orders); every repetition
must equal the first bit for bit."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REPS = 6


def _noise():
    """Background load on a second stream: HBM-bound copies."""
    import torch

    s = torch.cuda.Stream()
    a = torch.empty(1 << 27, dtype=torch.float32, device="cuda")
    b = torch.empty_like(a)
    with torch.cuda.stream(s):
        for _ in range(8):
            b.copy_(a)
    return s


def _ensemble_run(nx, nv, B, steps, hint=0):
    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs
    from paper_2511_13386_b200.engine import Device, HybridKnobs, make_phase

    cases = configs.cfg5(range(B), nx=nx, nv=nv)
    m = cases[0].mesh
    dev = Device.for_mesh(m)
    eps = [c.eps for c in cases]
    dts = [pk.kinetic.stable_dt(m, c.eps, e_max=float(np.abs(
        pk.solve_field(c.rho, c.rho_bar, m)).max())) for c in cases]
    ph = [make_phase(m, eps, dts, [steps] * B), make_phase(m, eps, dts, [0] * B)]
    rb = dev.t(np.array([c.rho_bar for c in cases]))
    outs = []
    for r in range(REPS):
        rho = dev.t(np.stack([c.rho for c in cases]))
        g = dev.t(np.stack([c.g.reshape(nx, nv) for c in cases]))
        E, Ep = torch.zeros_like(rho), torch.zeros_like(rho)
        kc = torch.ones((B, nx), dtype=torch.uint8, device=dev.device)
        ki = torch.ones_like(kc)
        s = _noise() if r % 2 else None
        dev.fine(rho, E, Ep, kc, ki, g, rb, [0] * B, ph, HybridKnobs(), eps, 1e-10,
                 cluster_hint=hint)
        dev.check()
        if s is not None:
            s.synchronize()
        outs.append((rho.cpu().numpy(), E.cpu().numpy(), g.cpu().numpy(), dev.last_launch()))
    return outs


@pytest.mark.parametrize("nx,nv,B,hint,kind", [(256, 128, 256, 0, 1),   # software groups
                                               (128, 64, 200, 0, 0),    # packed clusters
                                               (512, 128, 16, 0, 0),    # one slice per cluster
                                               (64, 256, 40, 0, None),   # nv = 256 layout
                                               (256, 128, 256, 1, 0)])   # one CTA per slice
def test_layouts_repeat_bitwise(nx, nv, B, hint, kind):
    outs = _ensemble_run(nx, nv, B, 12, hint)
    if kind is not None and "PK_NO_SG" not in os.environ:
        assert outs[0][3][3] == kind, outs[0][3]
    for o in outs[1:]:
        for a, b in zip(o[:3], outs[0][:3]):
            assert np.array_equal(a, b)


def _hybrid_cfg4_repeats(out_path):
    """cfg4 grid (8192 x 256): global-memory slice phase on every CTA of the
    cluster, 8 lifted windows, 16 hybrid steps, repeated under noise."""
    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs

    c = configs.cfg4()
    m = c.mesh
    E0 = pk.solve_field(c.rho, c.rho_bar, m, rtol=1e-5)
    g1 = pk.lift(c.rho, E0, c.eps, m, order=2, time_elim="leading", rho_bar=c.rho_bar)
    cfg = pk.PararealConfig(eps=c.eps, t_final=1.0, ng=8, thresholds=pk.Thresholds(1e-3, 1e-3))
    _, kin_p = pk.parareal.default_params(cfg, m, E0)
    st = pk.HybridState.initial(pk.MacroState(c.rho, E0, 0.0), g1, m)
    res = []
    for r in range(4):
        s = _noise() if r % 2 else None
        out = pk.hybrid_propagate(st, 16 * kin_p.dt, kin_p, pk.Thresholds(1e-3, 1e-3),
                                  pk.HybridOptions(), m, c.rho_bar, field_rtol=1e-5)
        if s is not None:
            s.synchronize()
        res.append(np.concatenate([out.macro.rho, out.macro.E,
                                   out.labels.kinetic_cells.astype(float),
                                   out.micro.g.reshape(-1)[::97]]))
    np.save(out_path, np.stack(res))


def test_hybrid_global_slice_repeat_bitwise(tmp_path):
    _hybrid_cfg4_repeats(tmp_path / "a.npy")
    r = np.load(tmp_path / "a.npy")
    for k in range(1, r.shape[0]):
        assert np.array_equal(r[k], r[0])


@pytest.mark.parametrize("mode", ["1", "2"])
def test_forced_global_slice_small_hybrid_repeat(mode, tmp_path):
    """PK_FORCE_GLOBAL_SLICE (test hook, read once per process): the same
    global-memory slice-phase protocols on a small hybrid golden case."""
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import test_determinism as T\n"
        "import paper_2511_13386_b200 as pk\n"
        "m = pk.build_mesh(pk.MeshSpec(nx=48, nvx=16))\n"
        "x = m.x_centers; rho = 1.0 + 0.5 * np.cos(x); rb = float(rho.sum() * m.dx / m.x_star)\n"
        "E0 = pk.solve_field(rho, rb, m)\n"
        "g = pk.lift(rho, E0, 0.5, m, order=2, time_elim='leading', rho_bar=rb)\n"
        "p = pk.KineticStepParams.default(m, 1e-2, e_max=float(np.abs(E0).max()))\n"
        "st = pk.HybridState.initial(pk.MacroState(rho, E0, 0.0), g, m)\n"
        "res = []\n"
        "for r in range(%d):\n"
        "    s = T._noise() if r %% 2 else None\n"
        "    o = pk.hybrid_propagate(st, 60 * p.dt, p, pk.Thresholds(1e-3, 1e-3), pk.HybridOptions(), m, rb, field_rtol=1.0)\n"
        "    s is not None and s.synchronize()\n"
        "    res.append(np.concatenate([o.macro.rho, o.macro.E, o.micro.g.reshape(-1), o.labels.kinetic_cells]))\n"
        "np.save(%r, np.stack(res))\n" % (ROOT, os.path.join(ROOT, "tests"), REPS,
                                          str(tmp_path / "r.npy")))
    env = dict(os.environ, PK_FORCE_GLOBAL_SLICE=mode)
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    r = np.load(tmp_path / "r.npy")
    for k in range(1, r.shape[0]):
        assert np.array_equal(r[k], r[0])


def test_big_rows_repeat_bitwise():
    """The reference's default 32 x 16 x 16 grid, one CTA per row."""
    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200.ensemble import Ensemble

    nx = 32
    m = pk.build_mesh(pk.MeshSpec(nx=nx, nvx=32, nvy=16, nvz=16))
    grid = m.vgrid
    w = grid.xi**4 * grid.M
    f = lambda x: w[None] * (1.0 + 0.9 * np.cos(2.0 * np.pi * x / m.x_star))[:, None, None, None]  # noqa: E731
    rho = m.bracket_x(f(m.x_centers))
    f_if = f(m.x_interfaces)
    g0 = f_if - m.bracket_x(f_if)[:, None, None, None] * grid.M[None]
    rb = float(rho.sum() * m.dx / m.x_star)
    E0 = pk.solve_field(rho, rb, m)
    p = pk.KineticStepParams.default(m, 0.5, e_max=float(np.abs(E0).max()))
    B = 12
    ens = Ensemble(m, [0.5] * B, [p.dt] * B, [rb] * B)
    outs = []
    for r in range(REPS):
        ens.load(np.tile(rho, (B, 1)), np.tile(g0.reshape(1, nx, -1), (B, 1, 1)))
        s = _noise() if r % 2 else None
        ens.run(6)
        if s is not None:
            s.synchronize()
        outs.append((ens.rho.cpu().numpy(), ens.g.cpu().numpy()))
        torch.cuda.synchronize()
    assert ens.dev.last_launch()[3] in (2, 3) or "PK_NO_BIGC" in os.environ
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])
