"""Profiling driver for the fine kernel: cfg5-type ensemble, configurable size.

  python tools/prof_fine.py --B 256 --steps 20 [--reps 2] [--nx 1024 --nv 128] [--per-cta]

Prints per-launch CUDA-event times; meant to be wrapped by ncu (-k regex:fine_kernel).
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=256)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--nx", type=int, default=1024)
    ap.add_argument("--nv", type=int, default=128)
    ap.add_argument("--per-cta", action="store_true")
    a = ap.parse_args()
    import torch

    from paper_2511_13386_b200 import configs
    from paper_2511_13386_b200.ensemble import Ensemble
    from paper_2511_13386_b200.kinetic import stable_dt
    from paper_2511_13386_b200.poisson import solve_field

    cases = configs.cfg5(range(a.B), nx=a.nx, nv=a.nv)
    m = cases[0].mesh
    dts = []
    for c in cases:
        E0 = solve_field(c.rho, c.rho_bar, m)
        dts.append(stable_dt(m, c.eps, e_max=float(np.abs(E0).max())))
    ens = Ensemble(m, [c.eps for c in cases], dts, [c.rho_bar for c in cases])
    rho = torch.from_numpy(np.stack([c.rho for c in cases])).cuda()
    g = torch.from_numpy(np.stack([c.g.reshape(a.nx, a.nv) for c in cases])).cuda()
    cnt = torch.zeros(32 + 3 * 1024, dtype=torch.int64, device="cuda")
    ens.dev.lib.pk_debug_profile(ens.dev.ctx, cnt.data_ptr())
    for r in range(a.reps):
        cnt.zero_()
        ens.load(rho, g)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ens.run(a.steps)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        upd = a.B * a.steps * a.nx * a.nv
        print(f"rep {r}: {ms:.3f} ms, {ms / a.steps * 1e3:.1f} us/step, "
              f"{upd / ms * 1e3:.3e} cell-updates/s, {16 * upd / ms / 1e6:.1f} GB/s alg")
        c = cnt.cpu().numpy()
        ns = max(int(c[5]), 1)
        print("   slice0 cycles/step: micro %d, bar %d, finish %d, prepare %d, bar %d"
              % tuple(int(x) // ns for x in c[:5]))
        print("   field cycles/step: src %d, pairwise2 %d, corr %d, cumsum %d, mean %d, sub %d"
              % tuple(int(x) // ns for x in c[8:14]))
        print("   slice vectors in shared memory:", bool(c[15]))
        C, K, _, sg = ens.dev.last_launch()
        print(f"   launch: {'software groups' if sg == 1 else 'clusters'} of {C} CTAs x {K} slices")
        if a.per_cta:
            ncta = (a.B + K - 1) // K * C
            pc = c[32:32 + 3 * ncta].reshape(ncta, 3)
            mic, bar = pc[:, 0] / ns, pc[:, 1] / ns
            print("   per-CTA micro cycles/step: min %d median %d max %d; first-barrier wait "
                  "min %d median %d max %d" % (mic.min(), np.median(mic), mic.max(), bar.min(),
                                               np.median(bar), bar.max()))
            per_sm = np.bincount(pc[:, 2], minlength=148)
            for r in range(C):  # by rank within the group
                sel = np.arange(ncta) % C == r
                print(f"     rank {r}: micro median {np.median(mic[sel]):.0f} max "
                      f"{mic[sel].max():.0f}, bar median {np.median(bar[sel]):.0f}, "
                      f"SM-mates {np.mean(per_sm[pc[sel, 2]]):.2f}")
            grp = np.arange(ncta) // C
            gmax = np.array([mic[grp == q].max() for q in range(grp.max() + 1)])
            gmin = np.array([mic[grp == q].min() for q in range(grp.max() + 1)])
            print("   per-group micro max: min %d median %d max %d; spread (max-min) median %d"
                  % (gmax.min(), np.median(gmax), gmax.max(), np.median(gmax - gmin)))
            for nmate in (1, 2):
                sel = per_sm[pc[:, 2]] == nmate
                if sel.any():
                    print(f"     CTAs on SMs holding {nmate}: {sel.sum()}, micro median "
                          f"{np.median(mic[sel]):.0f}")


if __name__ == "__main__":
    main()
