"""Per-step time of the coarse propagator G (chain_kernel) through the drop-in
fluid_propagate: cfg4's nx = 8192 and cfg2's nx = 256 (one chain, one window,
n steps at the reference coarse dt), CUDA events around the call.

  python tools/coarse_step.py [--steps 2000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2000)
    a = ap.parse_args()
    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs

    for name, c in (("cfg4", configs.cfg4()), ("cfg2", configs.cfg2())):
        m = c.mesh
        p = pk.FluidStepParams.default(m)
        E0 = pk.solve_field(c.rho, c.rho_bar, m)
        st = pk.MacroState(c.rho, E0, 0.0)
        t_end = a.steps * p.dt
        pk.fluid_propagate(st, 10 * p.dt, p, m, c.rho_bar)  # warm-up
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pk.fluid_propagate(st, t_end, p, m, c.rho_bar)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            print(f"{name} nx={m.nx}: {a.steps} coarse steps in {dt * 1e3:.1f} ms = "
                  f"{dt / a.steps * 1e6:.2f} us per step (host wall around one chain launch)")


if __name__ == "__main__":
    main()
