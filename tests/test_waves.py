"""Residency of persistent cluster launches: a grid whose hardware
clusters are not all co-resident runs in waves, each a whole launch long.  The
launcher sizes clusters from the measured residency table; the results must
not depend on the cluster size, and a launch that would have needed a second
wave must come out with a size that fits."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _hybrid_batch(nx, nv, B, steps, hint=0):
    import torch  # noqa: F401

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200.engine import Device, make_phase

    m = pk.build_mesh(pk.MeshSpec(nx=nx, nvx=nv))
    x = m.x_centers
    rho = 1.0 + 0.5 * np.cos(x)
    rb = float(rho.sum() * m.dx / m.x_star)
    E0 = pk.solve_field(rho, rb, m)
    eps = 0.05
    p = pk.KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
    dev = Device.for_mesh(m)
    knobs = pk.hybrid.knobs_of(pk.HybridOptions(adaptation=True), pk.Thresholds(1e-3, 1e-3))
    phases = [make_phase(m, [eps] * B, [p.dt] * B, [steps] * B),
              make_phase(m, [eps] * B, [p.dt] * B, [0] * B)]
    r = dev.t(np.tile(rho, (B, 1)))
    E = dev.t(np.tile(E0, (B, 1)))
    Ep = E.clone()
    kc = dev.t(np.ones((B, nx), dtype=np.uint8))
    ki = kc.clone()
    g = dev.t(np.zeros((B, nx, nv)))
    rbt = dev.t(np.full(B, rb))
    # a window restart: g := lift(rho, E), E_prev := E
    dev.fine(r, E, Ep, kc, ki, g, rbt, [3] * B, phases, knobs, [eps] * B, 1e-5, cluster_hint=hint)
    dev.check()
    return (r.cpu().numpy(), E.cpu().numpy(), g.cpu().numpy(), ki.cpu().numpy(),
            dev.last_launch())


def test_hybrid_clusters_fit_one_wave():
    """37 hybrid slices of 1024 cells keep their vectors on chip at one CTA per
    SM; 37 clusters of 4 CTAs are not co-resident on a B200 (GPC packing: 33).
    The launch must pick a size whose clusters are, and every slice must equal
    the single-slice launch bit for bit."""
    nx, nv, B, steps = 1024, 64, 37, 6
    one = _hybrid_batch(nx, nv, 1, steps)
    many = _hybrid_batch(nx, nv, B, steps)
    C, K, on_chip, kind = many[4]
    assert kind == 0 and K == 1
    if on_chip:  # one CTA per SM: at most 33 clusters of 4, 45 of 3 are resident
        assert B * C <= 148 and C <= 3, many[4]
    for k in range(B):
        for a, b in zip(many[:4], one[:4]):
            assert np.array_equal(a[k], b[0])
    # and independent of an explicit cluster size
    two = _hybrid_batch(nx, nv, 5, steps, hint=2)
    for a, b in zip(two[:4], one[:4]):
        assert np.array_equal(a[0], b[0])


@pytest.mark.skipif("PK_NO_CANCEL" in __import__("os").environ, reason="A/B switch: cancel disabled")
def test_fine_cancel_stops_a_window():
    """pk_fine_cancel: a window launched for far more steps than needed (the
    overlapped parareal schedule's speculative windows) stops at its next step
    when asked, and the context runs the next launch normally."""
    import time

    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200.engine import Device, make_phase

    nx, nv = 256, 64
    m = pk.build_mesh(pk.MeshSpec(nx=nx, nvx=nv))
    rho = 1.0 + 0.3 * np.cos(m.x_centers)
    rb = float(rho.sum() * m.dx / m.x_star)
    E0 = pk.solve_field(rho, rb, m)
    eps = 1e-2
    p = pk.KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
    dev = Device.for_mesh(m)
    knobs = pk.hybrid.knobs_of(pk.HybridOptions(adaptation=False), pk.Thresholds(1e-3, 1e-3))

    def launch(steps):
        phases = [make_phase(m, [eps], [p.dt], [steps]), make_phase(m, [eps], [p.dt], [0])]
        r = dev.t(rho[None].copy())
        E = dev.t(E0[None].copy())
        Ep = E.clone()
        kc = dev.t(np.ones((1, nx), dtype=np.uint8))
        ki = kc.clone()
        g = dev.t(np.zeros((1, nx, nv)))
        dev.fine(r, E, Ep, kc, ki, g, dev.t(np.full(1, rb)), [3], phases, knobs, [eps], 1e-5)
        return r, g

    ref_r, ref_g = launch(50)
    dev.check()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    t0 = time.perf_counter()
    launch(200000)               # ~1.5 s of steps if left alone
    time.sleep(0.02)
    dev.cancel(side)
    torch.cuda.synchronize()
    assert time.perf_counter() - t0 < 0.5
    dev.check()                  # a cancelled launch latches no error
    r, g = launch(50)            # the request was for that launch only
    dev.check()
    assert np.array_equal(r.cpu().numpy(), ref_r.cpu().numpy())
    assert np.array_equal(g.cpu().numpy(), ref_g.cpu().numpy())
