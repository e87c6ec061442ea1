"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck) through
every launch layout of libpk: hardware clusters (one slice each, packed K < C),
software groups (cooperative launch, moments through global memory with
signalling-NaN sentinels and counter barriers), the nv = 256 producer/consumer
layout, big 1D-3V rows (one CTA per row, and one warp per row), the hybrid
slice phase on chip and -- with PK_FORCE_GLOBAL_SLICE=1|2 in the environment
-- in global memory, the coarse chain (exact and fast scan), lift, field,
jump and maxdiff.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py --case sg

Every case checks its launch layout and the device status; results are
checked for parity by the test suite, not here.
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def ensemble(nx, nv, B, steps, want_kind=None, hint=0):
    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs
    from paper_2511_13386_b200.engine import HybridKnobs, make_phase

    cases = configs.cfg5(range(B), nx=nx, nv=nv)
    m = cases[0].mesh
    dev = pk.engine.Device.for_mesh(m)
    eps = [c.eps for c in cases]
    dts = []
    for c in cases:
        E0 = pk.solve_field(c.rho, c.rho_bar, m)
        dts.append(pk.kinetic.stable_dt(m, c.eps, e_max=float(np.abs(E0).max())))
    import torch

    rho = dev.t(np.stack([c.rho for c in cases]))
    g = dev.t(np.stack([c.g.reshape(nx, nv) for c in cases]))
    E, Ep = torch.zeros_like(rho), torch.zeros_like(rho)
    kc = torch.ones((B, nx), dtype=torch.uint8, device=dev.device)
    ki = torch.ones_like(kc)
    ph = [make_phase(m, eps, dts, [steps] * B), make_phase(m, eps, dts, [0] * B)]
    dev.fine(rho, E, Ep, kc, ki, g, dev.t(np.array([c.rho_bar for c in cases])), [0] * B, ph,
             HybridKnobs(), eps, 1e-10, cluster_hint=hint)
    dev.check()
    lay = dev.last_launch()
    print("layout (C, K, on_chip, kind):", lay)
    if want_kind is not None:
        assert lay[3] == want_kind, lay


def hybrid(nx, nv, steps, eps=1e-2, th=1e-3):
    import paper_2511_13386_b200 as pk

    m = pk.build_mesh(pk.MeshSpec(nx=nx, nvx=nv))
    x = m.x_centers
    rho = 1.0 + 0.5 * np.cos(x)
    rb = float(rho.sum() * m.dx / m.x_star)
    E0 = pk.solve_field(rho, rb, m)
    g = pk.lift(rho, E0, 0.5, m, order=2, time_elim="leading", rho_bar=rb)
    p = pk.KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
    st = pk.HybridState.initial(pk.MacroState(rho, E0, 0.0), g, m)
    out = pk.hybrid_propagate(st, steps * p.dt, p, pk.Thresholds(th, th), pk.HybridOptions(), m,
                              rb, field_rtol=1.0)
    print("kinetic fraction", out.labels.kinetic_fraction)


def v3(nvx, nvy, nvz, nx=8, steps=2):
    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200.ensemble import Ensemble

    m = pk.build_mesh(pk.MeshSpec(nx=nx, nvx=nvx, nvy=nvy, nvz=nvz))
    grid = m.vgrid
    w = grid.xi**4 * grid.M
    f = lambda x: w[None] * (1.0 + 0.9 * np.cos(2.0 * np.pi * x / m.x_star))[:, None, None, None]  # noqa: E731
    rho = m.bracket_x(f(m.x_centers))
    f_if = f(m.x_interfaces)
    g0 = f_if - m.bracket_x(f_if)[:, None, None, None] * grid.M[None]
    rb = float(rho.sum() * m.dx / m.x_star)
    E0 = pk.solve_field(rho, rb, m)
    p = pk.KineticStepParams.default(m, 0.5, e_max=float(np.abs(E0).max()))
    ens = Ensemble(m, [0.5] * 2, [p.dt] * 2, [rb] * 2)
    ens.load(np.tile(rho, (2, 1)), np.tile(g0.reshape(1, nx, -1), (2, 1, 1)))
    ens.run(steps)
    print("layout:", ens.dev.last_launch())
    # and a hybrid window on the same grid
    st = pk.HybridState.initial(pk.MacroState(rho, E0, 0.0), pk.MicroState(g0), m)
    pk.hybrid_propagate(st, steps * p.dt, p, pk.Thresholds(1.0, 1.0),
                        pk.HybridOptions(combine="and"), m, rb, field_rtol=1.0)


def chain_ops():
    import paper_2511_13386_b200 as pk

    for nx in (256, 3000):
        m = pk.build_mesh(pk.MeshSpec(nx=nx, nvx=8))
        x = m.x_centers
        rho = 1.0 + 0.3 * np.cos(x)
        rb = float(rho.sum() * m.dx / m.x_star)
        p = pk.FluidStepParams.default(m)
        E0 = pk.solve_field(rho, rb, m)
        for exact in (True, False):
            with pk.scan_mode(exact):
                pk.fluid_propagate(pk.MacroState(rho, E0, 0.0), 20.5 * p.dt, p, m, rb)
                pk.fluid_step(pk.MacroState(rho, E0, 0.0), p, m, rb)
                pk.solve_field(rho, rb, m)
        pk.lift(rho, E0, 0.1, m, order=2, time_elim="higher_order", rho_bar=rb)


def parareal_small():
    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs

    c = configs.cfg2(nx=64, nv=16)
    cfg = pk.PararealConfig(eps=1e-2, t_final=0.05, ng=4, k_max=3, tol=1e-10,
                            options=pk.HybridOptions(adaptation=False))
    res = pk.run(cfg, c.rho, c.g, c.mesh, c.rho_bar)   # overlapped schedule, jump/maxdiff
    print(res.status, res.iterations)


CASES = {
    "cluster": lambda: ensemble(64, 64, 4, 6, want_kind=0),
    "cluster128": lambda: ensemble(64, 128, 4, 6, want_kind=0),
    "packed": lambda: ensemble(32, 64, 170, 3),
    "sg": lambda: ensemble(256, 128, 256, 3, want_kind=1),
    "single": lambda: ensemble(64, 64, 3, 4, hint=1),
    "nv256": lambda: ensemble(64, 256, 3, 4),
    "generic": lambda: ensemble(24, 200, 3, 4),
    "hybrid": lambda: hybrid(48, 16, 40),
    "hybrid128": lambda: hybrid(64, 128, 30, eps=1e-3, th=1e-2),
    "hybrid256": lambda: hybrid(64, 256, 20, eps=1e-3, th=1e-2),
    "bigc": lambda: v3(32, 16, 16),
    "bigw": lambda: v3(17, 8, 8),
    "v3small": lambda: v3(8, 4, 4, nx=16, steps=4),
    "chain": chain_ops,
    "parareal": parareal_small,
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", choices=sorted(CASES) + ["all"], default="all")
    a = ap.parse_args()
    for name in (sorted(CASES) if a.case == "all" else [a.case]):
        print("case", name, flush=True)
        CASES[name]()
    import torch

    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
