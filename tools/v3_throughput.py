"""Fine-solver throughput on 1D-3V grids (the big-row path beyond 256 velocity
nodes), B instances of the paper recipe through the ensemble API.

  python tools/v3_throughput.py [--nx 256 --nvx 32 --nvy 16 --nvz 16 --B 16 --steps 50]
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=256)
    ap.add_argument("--nvx", type=int, default=32)
    ap.add_argument("--nvy", type=int, default=16)
    ap.add_argument("--nvz", type=int, default=16)
    ap.add_argument("--B", type=int, default=16)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200.ensemble import Ensemble

    m = pk.build_mesh(pk.MeshSpec(nx=a.nx, nvx=a.nvx, nvy=a.nvy, nvz=a.nvz))
    grid = m.vgrid
    w = grid.xi**4 * grid.M

    def f(x):
        return w[None] * (1.0 + 0.9 * np.cos(2.0 * np.pi * x / m.x_star))[:, None, None, None]

    rho = m.bracket_x(f(m.x_centers))
    f_if = f(m.x_interfaces)
    g0 = f_if - m.bracket_x(f_if)[:, None, None, None] * grid.M[None]
    rb = float(rho.sum() * m.dx / m.x_star)
    E0 = pk.solve_field(rho, rb, m)
    p = pk.KineticStepParams.default(m, 0.5, e_max=float(np.abs(E0).max()))
    ens = Ensemble(m, [0.5] * a.B, [p.dt] * a.B, [rb] * a.B)
    rho_d = torch.from_numpy(np.tile(rho, (a.B, 1))).cuda()
    g_d = torch.from_numpy(np.tile(g0.reshape(1, a.nx, -1), (a.B, 1, 1))).cuda()
    cnt = torch.zeros(32 + 3 * 1024, dtype=torch.int64, device="cuda")
    ens.dev.lib.pk_debug_profile(ens.dev.ctx, cnt.data_ptr())
    for rep in range(a.reps):
        cnt.zero_()
        ens.load(rho_d, g_d)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ens.run(a.steps)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        upd = a.B * a.steps * a.nx * m.nv
        print(f"rep {rep}: {ms:.2f} ms, {upd / ms * 1e3:.3e} cell-updates/s, "
              f"{16 * upd / ms / 1e6:.0f} GB/s algorithmic (grid {a.nx} x {a.nvx}x{a.nvy}x{a.nvz}, "
              f"B={a.B}, {a.steps} steps)")
        c = cnt.cpu().numpy()
        ns = max(int(c[5]), 1)
        print("   slice0 cycles/step: micro %d, bar %d, finish %d, prepare %d, bar %d"
              % tuple(int(x) // ns for x in c[:5]))
        print("   launch (CTAs per cluster, slices per cluster, on chip, group/bigc):",
              ens.dev.last_launch())


if __name__ == "__main__":
    main()
