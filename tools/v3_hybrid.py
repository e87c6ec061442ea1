"""Hybrid (adaptation on) fine windows on the reference's default 1D-3V grid
(32x16x16 velocity nodes) with cfg3's eps(x) profile: B window restarts
(g := lift(rho, E)), the big-row one-CTA-per-row layout on listed rows.

  python tools/v3_hybrid.py [--nx 128 --B 37 --steps 100]
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=128)
    ap.add_argument("--B", type=int, default=37)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--thr", type=float, default=1e-3)
    a = ap.parse_args()
    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs
    from paper_2511_13386_b200.configs import EpsProfile
    from paper_2511_13386_b200.engine import Device, make_phase

    m = pk.build_mesh(pk.MeshSpec(nx=a.nx, nvx=32, nvy=16, nvz=16))
    nx, nv = m.nx, m.nv
    rho = 1.0 + 0.5 * np.cos(m.x_centers)
    rb = float(rho.sum() * m.dx / m.x_star)
    E0 = pk.solve_field(rho, rb, m)
    eps = EpsProfile.from_function(configs.eps_bump, m)
    cfg = pk.PararealConfig(eps=eps, t_final=1.0, ng=8, thresholds=pk.Thresholds(a.thr, a.thr))
    _, kin_p = pk.parareal.default_params(cfg, m, E0)
    dev = Device.for_mesh(m)
    knobs = pk.hybrid.knobs_of(pk.HybridOptions(adaptation=True), pk.Thresholds(a.thr, a.thr))
    B = a.B
    phases = [make_phase(m, [eps] * B, [kin_p.dt] * B, [a.steps] * B),
              make_phase(m, [eps] * B, [kin_p.dt] * B, [0] * B)]
    cnt = torch.zeros(32 + 3 * 1024, dtype=torch.int64, device="cuda")
    dev.lib.pk_debug_profile(dev.ctx, cnt.data_ptr())
    rows = torch.zeros((B, 2), dtype=torch.int64, device="cuda")
    for r in range(a.reps):
        rh = dev.t(np.tile(rho, (B, 1)))
        E = dev.t(np.tile(E0, (B, 1)))
        Ep = E.clone()
        kc = dev.t(np.ones((B, nx), dtype=np.uint8))
        ki = kc.clone()
        g = dev.t(np.zeros((B, nx, nv)))
        rbt = dev.t(np.full(B, rb))
        dev.scratch("gb", (B, nx, nv))
        cnt.zero_()
        rows.zero_()
        dev.lib.pk_count_rows(dev.ctx, rows.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.fine(rh, E, Ep, kc, ki, g, rbt, [3] * B, phases, knobs, [eps] * B, 1e-2)
        e1.record()
        torch.cuda.synchronize()
        dev.lib.pk_count_rows(dev.ctx, None)
        ms = e0.elapsed_time(e1)
        try:
            dev.check()
        except Exception as e:  # noqa: BLE001
            print("status:", e)
        kin_rows = int(rows[:, 0].sum().item())
        print(f"rep {r}: {ms:.2f} ms, {ms / a.steps * 1e3:.1f} us/step, kinetic rows streamed "
              f"{kin_rows} ({kin_rows / (B * a.steps * nx):.3f} of all), "
              f"{kin_rows * nv / ms * 1e3:.3e} kinetic cell-updates/s = "
              f"{16 * kin_rows * nv / ms / 1e6:.0f} GB/s algorithmic; layout {dev.last_launch()}")
        cc = cnt.cpu().numpy()
        ns = max(int(cc[5]), 1)
        print("   slice0 cycles/step: micro %d, bar %d, finish %d, prepare %d, bar %d; prologue %d"
              % (tuple(int(x) // ns for x in cc[:5]) + (int(cc[6]),)))


if __name__ == "__main__":
    main()
