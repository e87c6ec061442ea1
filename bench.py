#!/usr/bin/env python
"""Benchmark: micro-macro phase-space cell-updates/s of the fine solver F.

Workload (BASELINE.json configs[4], the largest single-GPU throughput config):
256 seeded instances, Nx=1024, Nv=128, eps log-uniform in [1e-4, 1], 500
kinetic steps each at the reference's stable dt.  One bench "step" = one pass
of the hot path over the whole batch (256 x 500 x 1024 x 128 = 1.68e10
cell-updates).  Under torchrun the instances are partitioned across ranks
(strong scaling, no data-path collective).  Also reported: cfg2 parareal wall
time (BASELINE configs[1]) on this GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import os

# before any CUDA context exists (see paper_2511_13386_b200/__init__.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "micro-macro cell-updates/s (fine solver)"
UNIT = "cell-updates/s"
NINST, NX, NV, NSTEPS = 256, 1024, 128, 500
BYTES_PER_UPDATE = 16  # read g once, write g once, fp64


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons, sampled every 50 ms from before the
    warm-up to after the timed region; `summary(t0, t1)` keeps the samples whose
    host timestamps fall inside the timed region (nvidia-smi takes a few hundred
    ms to start, so starting it at the timed region could miss a short one)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def wait_first(self, timeout=5.0):
        t_end = time.perf_counter() + timeout
        while self.proc and not self.rows and time.perf_counter() < t_end:
            time.sleep(0.01)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if self.proc:
            time.sleep(0.06)  # let the sample covering the region's end arrive
            self.proc.terminate()
            self.proc.wait()

    def summary(self, t0, t1):
        rows = [r for t, r in self.rows if t0 <= t <= t1 + 0.06]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[2:6]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def build_inputs(instances):
    from paper_2511_13386_b200 import configs
    from paper_2511_13386_b200.kinetic import stable_dt
    from paper_2511_13386_b200.poisson import solve_field

    cases = configs.cfg5(instances, nx=NX, nv=NV)
    m = cases[0].mesh
    rho = np.stack([c.rho for c in cases])
    g = np.stack([c.g.reshape(NX, NV) for c in cases])
    eps = [c.eps for c in cases]
    rb = [c.rho_bar for c in cases]
    dts = []
    for c in cases:
        E0 = solve_field(c.rho, c.rho_bar, m)
        dts.append(stable_dt(m, c.eps, e_max=float(np.max(np.abs(E0)))))
    return m, cases, rho, g, eps, rb, dts


# ---------------------------------------------------------------------------
# CPU baseline: the oracle (numpy restatement of the reference, CPU port)


def _cpu_job(args):
    s, nsteps = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import oracle as O
    from paper_2511_13386_b200 import configs

    c = configs.cfg5([s], nx=NX, nv=NV)[0]
    grid = O.make_grid(NX, NV)
    E0 = O.field(c.rho, c.rho_bar, grid)
    dt = O.stable_dt(grid, c.eps, e_max=float(np.abs(E0).max()))
    g = c.g.reshape(NX, NV)
    t0 = time.perf_counter()
    O.kinetic_steps(c.rho, g, nsteps, dt, c.eps, grid, c.rho_bar)
    return time.perf_counter() - t0


def cpu_baseline(n_inst=None, nsteps=40):
    """Oracle on a bounded sample: one instance per process, all host cores."""
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    procs = min(cores, 64)
    n_inst = n_inst or procs
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(procs) as pool:
        pool.map(_cpu_job, [(s, nsteps) for s in range(n_inst)])
    wall = time.perf_counter() - t0
    upd = n_inst * nsteps * NX * NV
    return {"value": upd / wall, "unit": UNIT, "cores": procs, "kind": "port",
            "sample": f"{n_inst} cfg5 instances x {nsteps} steps (1024x128), one numpy "
                      f"process per instance, wall {wall:.2f} s incl. pool start"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    steps, warm = args.steps, args.warmup
    per = []
    for i in range(warm + steps):
        cb = cpu_baseline(nsteps=20)
        if i >= warm:
            per.append(cb["value"])
    v = statistics.median(per)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
            "steps": steps, "warmup": warm, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg5 ensemble: 256 x (1024x128), 500 kinetic steps; "
                                   "reference arm = oracle CPU port on a bounded sample"},
            "cpu_baseline": {**cb, "value": v},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parareal", action="store_true")
    ap.add_argument("--no-v3", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev_index = torch.cuda.current_device()

    from paper_2511_13386_b200.ensemble import Ensemble

    mine = list(range(NINST))[rank::ws] if ws > 1 else list(range(NINST))
    m, cases, rho0, g0, eps, rb, dts = build_inputs(mine)
    B = len(mine)
    ens = Ensemble(m, eps, dts, rb)
    rho_d = torch.from_numpy(rho0).cuda()
    g_d = torch.from_numpy(g0).cuda()
    upd_rank = B * NSTEPS * NX * NV

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def maxr(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    clk = ClockSampler(dev_index).start()
    clk.wait_first()
    # warm-up (untimed)
    for _ in range(args.warmup):
        ens.load(rho_d, g_d)
        ens.run(NSTEPS)
    barrier()
    # timed region: device-resident inputs (restored on device each step)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kstart = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    barrier()
    h0 = time.perf_counter()
    t0.record()
    for i in range(args.steps):
        starts[i].record()
        ens.load(rho_d, g_d)
        kstart[i].record()
        ens.run(NSTEPS, check=False)
        ends[i].record()
    t1.record()
    barrier()
    h1 = time.perf_counter()
    clk.stop()
    clocks = clk.summary(h0, h1)
    ens.dev.check()
    total_ms = maxr(t0.elapsed_time(t1))
    kern_ms = [kstart[i].elapsed_time(ends[i]) for i in range(args.steps)]
    kern_avg = maxr(sum(kern_ms) / len(kern_ms))
    ms_step = total_ms / args.steps
    value = upd_rank * ws * args.steps / (total_ms * 1e-3)
    peak, peak_src = peaks()
    achieved = upd_rank * BYTES_PER_UPDATE / (kern_avg * 1e-3) / 1e9

    # e2e: the public host-array streaming API (EnsemblePipeline): every step
    # uploads its inputs from pinned host memory and downloads rho, E and g;
    # uploads/downloads of neighbouring steps overlap the kernel
    from paper_2511_13386_b200.ensemble import EnsemblePipeline

    rho_h = torch.from_numpy(rho0).pin_memory()
    g_h = torch.from_numpy(g0).pin_memory()
    rho_o = torch.empty_like(rho_h).pin_memory()
    E_o = torch.empty_like(rho_h).pin_memory()
    g_o = torch.empty_like(g_h).pin_memory()
    pipe = EnsemblePipeline(m, eps, dts, rb, NSTEPS)
    for _ in range(2):  # warm-up of both state sets
        pipe.submit(rho_h, g_h, rho_o, E_o, g_o)
    pipe.drain()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(pipe.h2d)
    for _ in range(args.steps):
        pipe.submit(rho_h, g_h, rho_o, E_o, g_o)
    e1.record(pipe.d2h)
    pipe.drain()
    barrier()
    e2e_ms = maxr(e0.elapsed_time(e1))
    e2e = upd_rank * ws * args.steps / (e2e_ms * 1e-3)
    h2d = (rho_h.numel() + g_h.numel()) * 8 * ws
    d2h = (rho_o.numel() * 2 + g_o.numel()) * 8 * ws

    extra = {}
    if not args.no_parareal:
        # collective: every rank runs the engine (windows dealt across ranks)
        par = parareal_cfg2(barrier, maxr)
        if rank == 0:
            extra["parareal"] = par
    if rank == 0 and not args.no_v3:
        extra["v3"] = v3_default_grid(peak)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "fine_kernel_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f)
        if tr.get("nv") == NV and tr.get("nx") == NX:
            traffic = tr.get("bytes_per_launch")
    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg5 ensemble: 256 seeded instances x (Nx=1024, Nv=128), "
                                   "500 kinetic steps at the reference stable dt",
                       "instances": NINST, "nx": NX, "nv": NV, "steps_per_instance": NSTEPS,
                       "cell_updates_per_step": NINST * NSTEPS * NX * NV,
                       "parallelism": f"instances/{ws} per GPU" if ws > 1 else "1 GPU",
                       "l2": "inputs (2 x 256 MiB g buffers) larger than L2",
                       "mode": "exact (bitwise vs reference)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_src,
                         "traffic": traffic,
                         "algorithmic_bytes_per_update": BYTES_PER_UPDATE,
                         "kernel_ms": kern_avg},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
            **extra,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def parareal_cfg2(barrier, maxr):
    """BASELINE configs[1] through the drop-in run() on every rank (the engine
    deals the windows of each iteration across ranks and all-gathers the fine
    results).  Wall time = CUDA-event span on each rank's device timeline
    (host gaps between launches included), max over ranks."""
    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs

    c = configs.cfg2()
    cfg = pk.PararealConfig(eps=1e-2, t_final=0.5, ng=16, k_max=5, tol=1e-10,
                            options=pk.HybridOptions(adaptation=False))
    pk.run(cfg, c.rho, c.g, c.mesh, c.rho_bar)  # warm-up
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = pk.run(cfg, c.rho, c.g, c.mesh, c.rho_bar)
    e1.record()
    barrier()
    wall = maxr(e0.elapsed_time(e1) * 1e-3)
    tm = res.ledger.timings
    E0 = pk.solve_field(c.rho, c.rho_bar, c.mesh)
    _, kin_p = pk.parareal.default_params(cfg, c.mesh, E0)
    nf, rem = pk.fluid.substep_sizes(0.0, 0.5 / 16, kin_p.dt)
    per_window = (nf + (1 if rem > 0.0 else 0)) * 256 * 64
    fine_updates = sum(16 - k for k in range(res.iterations)) * per_window
    return {"config": "cfg2: Nx=256, Nv=64, eps=1e-2, T=0.5, 16 slices, reference dt",
            "wall_s": wall, "iterations": res.iterations, "status": res.status,
            "fine_s": maxr(tm.fine_total), "correction_s": maxr(tm.correction_total),
            "coarse_sweep_s": maxr(tm.coarse_sweep),
            "fine_cell_updates": fine_updates,
            "fine_cell_updates_per_s": fine_updates / max(tm.fine_total, 1e-12),
            "reference_cpu_s_build_container_1core": 41.7}


def v3_default_grid(peak, nx=128, B=37, steps=20):
    """The reference's own 1D-3V default velocity grid (32 x 16 x 16 nodes per
    interface), B seeded-recipe instances of nx cells through the ensemble API,
    all-kinetic steps at the reference stable dt: device-resident fine
    throughput (CUDA events around one launch of `steps` steps, after a
    warm-up launch) and its fraction of the HBM roofline at 16 B per update."""
    import numpy as np
    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200.ensemble import Ensemble

    m = pk.build_mesh(pk.MeshSpec(nx=nx, nvx=32, nvy=16, nvz=16))
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
    ens = Ensemble(m, [0.5] * B, [p.dt] * B, [rb] * B)
    rho_d = torch.from_numpy(np.tile(rho, (B, 1))).cuda()
    g_d = torch.from_numpy(np.tile(g0.reshape(1, nx, -1), (B, 1, 1))).cuda()
    ms = None
    for _ in range(2):
        ens.load(rho_d, g_d)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ens.run(steps)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    upd = B * steps * nx * m.nv
    val = upd / (ms * 1e-3)
    C, K, on_chip, layout = ens.dev.last_launch()
    return {"config": f"1D-3V default grid: {B} instances x Nx={nx} x (32x16x16) velocity nodes, "
                      f"{steps} kinetic steps, eps=0.5, device-resident",
            "value": val, "unit": "cell-updates/s", "ms": ms,
            "roofline_frac": val * 16 / (peak * 1e9),
            "layout": "one CTA per row" if layout == 2 else "warp per row"}


if __name__ == "__main__":
    main()
