"""Coarse propagator G at cfg4's nx = 8192: one fluid_propagate of --steps
coarse steps in exact mode (chain_kernel) and one in fast mode
(chain_fast_kernel), CUDA events around each (wrap in ncu -k regex:chain).

  python tools/prof_chain.py [--steps 500]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=500)
    a = ap.parse_args()
    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs

    c = configs.cfg4()
    m = c.mesh
    p = pk.FluidStepParams.default(m)
    E0 = pk.solve_field(c.rho, c.rho_bar, m)
    st = pk.MacroState(c.rho, E0, 0.0)
    for exact in (True, False):
        with pk.scan_mode(exact):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pk.fluid_propagate(st, a.steps * p.dt, p, m, c.rho_bar)
            e1.record()
            torch.cuda.synchronize()
            print(f"{'exact' if exact else 'fast'}: {e0.elapsed_time(e1) / a.steps * 1e3:.2f} us "
                  f"per coarse step (nx = {m.nx}, {a.steps} steps, host wall of one call)")


if __name__ == "__main__":
    main()
