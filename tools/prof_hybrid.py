"""Phase profile of the fine kernel on a hybrid (adaptation on) eps(x) case:
B copies of a lifted restart state (what parareal windows n >= 2 run).

  python tools/prof_hybrid.py --cfg 4 --B 8 --steps 20
  python tools/prof_hybrid.py --cfg 3 --B 32 --steps 200
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=4)
    ap.add_argument("--B", type=int, default=8)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--rtol", type=float, default=1e-5)
    ap.add_argument("--fast", action="store_true", help="fast scan mode (pk.scan_mode(False))")
    ap.add_argument("--hint", type=int, default=0, help="cluster size (0: the launcher's choice)")
    a = ap.parse_args()
    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs, engine
    from paper_2511_13386_b200.engine import Device, make_phase

    engine.EXACT = not a.fast

    c = configs.cfg4() if a.cfg == 4 else configs.cfg3()
    m = c.mesh
    nx, nv = m.nx, m.nv
    E0 = pk.solve_field(c.rho, c.rho_bar, m, rtol=a.rtol)
    cfg = pk.PararealConfig(eps=c.eps, t_final=1.0, ng=8, thresholds=pk.Thresholds(1e-3, 1e-3))
    _, kin_p = pk.parareal.default_params(cfg, m, E0)
    dev = Device.for_mesh(m)
    knobs = pk.hybrid.knobs_of(pk.HybridOptions(adaptation=True), pk.Thresholds(1e-3, 1e-3))
    phases = [make_phase(m, [c.eps] * a.B, [kin_p.dt] * a.B, [a.steps] * a.B),
              make_phase(m, [c.eps] * a.B, [kin_p.dt] * a.B, [0] * a.B)]
    cnt = torch.zeros(32 + 3 * 1024, dtype=torch.int64, device="cuda")
    dev.lib.pk_debug_profile(dev.ctx, cnt.data_ptr())
    for r in range(a.reps):
        rho = dev.t(np.tile(c.rho, (a.B, 1)))
        E = dev.t(np.tile(E0, (a.B, 1)))
        Ep = E.clone()
        kc = dev.t(np.ones((a.B, nx), dtype=np.uint8))
        ki = kc.clone()
        g = dev.t(np.zeros((a.B, nx, nv)))
        rb = dev.t(np.full(a.B, float(c.rho_bar)))
        prepared = dev.prepare_fine(a.B, phases, knobs, [c.eps] * a.B)
        dev.scratch("gb", (a.B, nx, nv))
        dev.reserve(a.B)
        cnt.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream())
        # bit0: lift g from (rho, E) at entry; bit1: E_prev := E (a window restart)
        dev.fine(rho, E, Ep, kc, ki, g, rb, [3] * a.B, phases, knobs, [c.eps] * a.B, a.rtol,
                 prepared=prepared, cluster_hint=a.hint)
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        try:
            dev.check()
        except Exception as e:  # noqa: BLE001
            print("status:", e)
        kf = ki.float().mean().item()
        upd = a.B * a.steps * nx * nv
        print(f"rep {r}: {ms:.2f} ms, {ms / a.steps * 1e3:.1f} us/step, kinetic-iface fraction "
              f"at end {kf:.3f}, {upd / ms * 1e3:.3e} nominal cell-updates/s")
        cc = cnt.cpu().numpy()
        ns = max(int(cc[5]), 1)
        print("   slice0 cycles/step: micro %d, bar %d, finish %d, prepare %d, bar %d"
              % tuple(int(x) // ns for x in cc[:5]))
        print("   field cycles/step: src %d, pairwise2 %d, corr %d, cumsum %d, mean %d, sub %d"
              % tuple(int(x) // ns for x in cc[8:14]))
        print("   prologue cycles: %d, slice vectors in shared memory: %s" % (int(cc[6]), bool(cc[15])))
        print("   prepare cycles/step: J %d, R+labels %d, flips %d, lift %d, bm %d, dco+zlist %d, "
              "zero %d, klist %d, kstream %d" % tuple(int(x) // ns for x in cc[16:25]))
        print("   rows/step: flipped %.1f, zeroed %.1f, kinetic %.1f"
              % tuple(float(x) / ns for x in cc[26:29]))
        print("   GS consumer warp 0 cycles/step: coefficients %d, waiting for rows %d, row operations %d"
              % tuple(int(x) // ns for x in cc[29:32]))
        Cc = dev.last_launch()[0]
        ncta = min(a.B * Cc, 1024)
        smid = [int(x) for x in cc[34:34 + 3 * ncta:3]]
        shared = len(smid) - len(set(smid))
        pm = [int(x) // ns for x in cc[32:32 + 3 * Cc:3]]
        pb = [int(x) // ns for x in cc[33:33 + 3 * Cc:3]]
        print(f"   slice 0 per-CTA cycles/step: micro {pm}, barrier after it {pb}")
        print(f"   clusters of {Cc}: {ncta} CTAs on {len(set(smid))} SMs ({shared} CTAs share an SM); "
              f"slice 0's CTAs on SMs {smid[:Cc]}")


if __name__ == "__main__":
    main()
