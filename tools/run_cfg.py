"""GPU runs of the epsilon(x) hybrid parareal configurations (BASELINE configs
3 and 4) through the drop-in API.

  python tools/run_cfg.py --cfg 3            # full run: Nx=512, Nv=128, 32 slices, T=1, tol 1e-8
  python tools/run_cfg.py --cfg 4 --fine-steps 200 --coarse-steps 50
      # Nx=8192, Nv=256, 64 slices: one parareal iteration at a reduced T
      # (each window shortened to `fine-steps` fine steps), per-step times
      # extrapolated to the full T = 2 window length

Prints one JSON object.  Synthetic inputs follow configs.py (seeded, as
BASELINE.json states); dt follows the reference rules.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def cfg3(args):
    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs

    c = configs.cfg3()
    th = pk.Thresholds(1e-3, 1e-3)
    cfg = pk.PararealConfig(eps=c.eps, t_final=1.0, ng=32, k_max=args.k_max, tol=1e-8,
                            thresholds=th, options=pk.HybridOptions(adaptation=True))
    E0 = pk.solve_field(c.rho, c.rho_bar, c.mesh)
    fluid_p, kin_p = pk.parareal.default_params(cfg, c.mesh, E0)
    nf, rem = pk.fluid.substep_sizes(0.0, 1.0 / 32, kin_p.dt)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = pk.run(cfg, c.rho, c.g, c.mesh, c.rho_bar)
    wall = time.perf_counter() - t0
    tm = res.ledger.timings
    steps = nf + (1 if rem > 0.0 else 0)
    windows = sum(32 - k for k in range(res.iterations))
    nominal = windows * steps * c.mesh.nx * c.mesh.nv
    kf = np.asarray(res.kinetic_fraction, dtype=float)
    mass = np.asarray(res.boundary_rho).sum(axis=1) * c.mesh.dx
    drift = float(np.max(np.abs(mass - mass[0])) / abs(mass[0]))
    return {"max_rel_mass_drift_boundary_rows": drift,"config": "cfg3: Nx=512, Nv=128, eps(x)=1e-3+0.5exp(-20(x-pi)^2), delta0=eta0=1e-3, "
                      "32 slices, T=1, tol 1e-8, reference dt",
            "status": res.status, "iterations": res.iterations, "err": [float(e) for e in res.ledger.err],
            "wall_s": wall, "fine_s": tm.fine_total, "correction_s": tm.correction_total,
            "coarse_sweep_s": tm.coarse_sweep, "fine_dt": kin_p.dt, "fine_steps_per_window": steps,
            "coarse_dt": fluid_p.dt,
            "nominal_cell_updates": nominal,
            "nominal_cell_updates_per_s_fine": nominal / max(tm.fine_total, 1e-12),
            "kinetic_fraction_mean": float(kf.mean()) if kf.size else None,
            "kinetic_fraction_min": float(kf.min()) if kf.size else None}


def cfg4(args):
    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs
    from paper_2511_13386_b200.engine import Device

    c = configs.cfg4()
    m = c.mesh
    th = pk.Thresholds(1e-3, 1e-3)
    T, ng = 2.0, 64
    cfg_full = pk.PararealConfig(eps=c.eps, t_final=T, ng=ng, k_max=1, tol=1e-8, thresholds=th,
                                 options=pk.HybridOptions(adaptation=True))
    E0 = pk.solve_field(c.rho, c.rho_bar, m, rtol=pk.parareal.ADAPTIVE_FIELD_RTOL)
    fluid_p, kin_p = pk.parareal.default_params(cfg_full, m, E0)
    nf_full, rem_full = pk.fluid.substep_sizes(0.0, T / ng, kin_p.dt)
    cf_full, crem_full = pk.fluid.substep_sizes(0.0, T / ng, fluid_p.dt)
    # reduced T: every window spans `fine_steps` fine steps exactly
    t_red = ng * args.fine_steps * kin_p.dt
    cfg = pk.PararealConfig(eps=c.eps, t_final=t_red, ng=ng, k_max=1, tol=1e-8, thresholds=th,
                            options=pk.HybridOptions(adaptation=True))
    # phase times from the phase-by-phase schedule (the overlapped one runs
    # the first iteration's windows during the coarse sweep), then the
    # overlapped wall time of the same sampled run
    walls = {}
    for ov in (False, True):
        pk.parareal.OVERLAP = ov
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = pk.run(cfg, c.rho, c.g, m, c.rho_bar)
        torch.cuda.synchronize()
        walls[ov] = time.perf_counter() - t0
        if not ov:
            res = r
    pk.parareal.OVERLAP = True
    wall = walls[False]
    tm = res.ledger.timings
    nf, rem = pk.fluid.substep_sizes(0.0, t_red / ng, kin_p.dt)
    steps = nf + (1 if rem > 0.0 else 0)
    fine_step_s = tm.fine_total / steps
    cnf, crem = pk.fluid.substep_sizes(0.0, t_red / ng, fluid_p.dt)
    csteps = cnf + (1 if crem > 0.0 else 0)
    # one coarse chain over all windows: time per coarse step
    dev = Device.for_mesh(m)
    rho = dev.t(np.ascontiguousarray(c.rho.reshape(1, -1)))
    out = dev.t(np.zeros((1, ng, m.nx)))
    nsteps = args.coarse_steps
    nfull = np.full((1, ng), nsteps, dtype=np.int32)
    remv = np.zeros((1, ng))
    rb = dev.t(np.array([float(c.rho_bar)]))
    for _ in range(2):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        dev.chain(rho, out, None, None, None, nfull, remv, fluid_p.dt, rb,
                  pk.parareal.ADAPTIVE_FIELD_RTOL, m2=fluid_p.m2)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        dev.check()
    coarse_step_s = (t2 - t1) / (ng * nsteps)
    full_steps = nf_full + (1 if rem_full > 0.0 else 0)
    full_csteps = cf_full + (1 if crem_full > 0.0 else 0)
    upd = ng * steps * m.nx * m.nv
    return {"config": "cfg4: Nx=8192, Nv=256, v*=10, eps(x) as cfg3, 64 slices on 1 GPU, "
                      "delta0=eta0=1e-3; one iteration at reduced T, extrapolated",
            "reduced_t_final": t_red, "fine_steps_per_window_sampled": steps,
            "status": res.status, "wall_s_sampled_iteration": wall,
            "wall_s_sampled_iteration_overlapped": walls[True],
            "fine_s_sampled": tm.fine_total, "fine_s_per_step_all_64_windows": fine_step_s,
            "nominal_cell_updates_per_s": upd / max(tm.fine_total, 1e-12),
            "coarse_s_per_step": coarse_step_s, "coarse_steps_per_window_sampled": csteps,
            "fine_dt": kin_p.dt, "coarse_dt": fluid_p.dt,
            "full_fine_steps_per_window": full_steps, "full_coarse_steps_per_window": full_csteps,
            "extrapolated_fine_s_per_iteration_1gpu": fine_step_s * full_steps,
            "extrapolated_fine_s_per_iteration_8gpu": fine_step_s * full_steps / 8,
            "extrapolated_coarse_sweep_s": coarse_step_s * full_csteps * ng,
            "kinetic_fraction_mean": float(np.mean(res.kinetic_fraction))
            if np.size(res.kinetic_fraction) else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, required=True, choices=(3, 4))
    ap.add_argument("--k-max", type=int, default=50)
    ap.add_argument("--fine-steps", type=int, default=200)
    ap.add_argument("--coarse-steps", type=int, default=50)
    ap.add_argument("--field-rtol", type=float, default=None,
                    help="relax the adaptive solvability guard (reference: 1e-5)")
    a = ap.parse_args()
    import paper_2511_13386_b200 as pk

    if a.field_rtol is not None:
        # explicit extension: the reference's module-level guard
        # (parareal.py:45-52) relaxed for the whole run, reported in the output
        pk.parareal.ADAPTIVE_FIELD_RTOL = a.field_rtol
    t0 = time.perf_counter()
    try:
        out = cfg3(a) if a.cfg == 3 else cfg4(a)
    except pk.SimulationError as e:  # the reference raises the same typed errors
        import traceback

        frames = [f"{fr.name}:{fr.lineno}" for fr in traceback.extract_tb(e.__traceback__)
                  if "paper_2511_13386_b200" in fr.filename]
        out = {"config": f"cfg{a.cfg}", "status": "raised", "error": type(e).__name__,
               "detail": str(e), "raised_in": frames[-4:],
               "wall_s_until_raise": time.perf_counter() - t0}
    out["field_rtol"] = pk.parareal.ADAPTIVE_FIELD_RTOL
    out["field_rtol_is_reference"] = a.field_rtol is None
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
