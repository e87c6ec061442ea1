#!/usr/bin/env python
"""Benchmark: micro-macro phase-space cell-updates/s of the fine solver F,
and parareal wall times.

Headline workload (BASELINE.json configs[4], the largest single-GPU throughput
config): 256 seeded instances, Nx=1024, Nv=128, eps log-uniform in [1e-4, 1],
500 kinetic steps each at the reference's stable dt.  One bench "step" = one
pass of the hot path over the whole batch (256 x 500 x 1024 x 128 = 1.68e10
cell-updates).  With N GPUs the instances are partitioned across ranks
(strong scaling, no data-path collective).  Extras on the same line:
parareal wall time of BASELINE cfg2 (configs[1]) and of a reduced-T cfg4
(configs[3]) iteration at N GPUs (windows dealt across ranks, NCCL
all-gather), BASELINE cfg3 (configs[2]) iteration 1 with its hybrid
fine-kernel roofline, the 1D-3V default grid, and the CPU path (the oracle
port of the reference) timed on this box's host cores.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--gpus N > 1 without a torchrun environment relaunches itself under
torch.distributed.run with N ranks (one per GPU).
"""

from __future__ import annotations

import os

# before any CUDA context exists (see paper_2511_13386_b200/__init__.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import argparse
import json
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


def workload_config(ws):
    """The `config` object of BOTH arms (same workload, same metric)."""
    return {"workload": "cfg5 ensemble: 256 seeded instances x (Nx=1024, Nv=128), "
                        "500 kinetic steps at the reference stable dt",
            "instances": NINST, "nx": NX, "nv": NV, "steps_per_instance": NSTEPS,
            "cell_updates_per_step": NINST * NSTEPS * NX * NV,
            "parallelism": f"instances/{ws} per GPU" if ws > 1 else "1 GPU",
            "l2": "inputs (2 x 256 MiB g buffers) larger than L2",
            "mode": "exact (bitwise vs reference)"}


# ---------------------------------------------------------------------------
# CPU path: the oracle (numpy restatement of the reference -- TEST
# INFRASTRUCTURE, used here only as the CPU baseline) on a pre-started process
# pool over the host cores.  Only the stepping itself is timed.


def _cpu_init():
    os.environ["OMP_NUM_THREADS"] = "1"
    import oracle  # noqa: F401
    from paper_2511_13386_b200 import configs  # noqa: F401


def _cpu_warm(_):
    import oracle as O

    O.make_grid(16, 8)
    return os.getpid()


def _cpu_cfg5(args):
    """One cfg5 instance: build (untimed), then `nsteps` kinetic steps.
    Returns the wall-clock interval of the stepping."""
    s, nsteps = args
    import oracle as O
    from paper_2511_13386_b200 import configs

    c = configs.cfg5([s], nx=NX, nv=NV)[0]
    grid = O.make_grid(NX, NV)
    E0 = O.field(c.rho, c.rho_bar, grid)
    dt = O.stable_dt(grid, c.eps, e_max=float(np.abs(E0).max()))
    g = c.g.reshape(NX, NV)
    t0 = time.time()
    with np.errstate(all="ignore"):
        O.kinetic_steps(c.rho, g, nsteps, dt, c.eps, grid, c.rho_bar)
    return t0, time.time()


def _cpu_cfg2_setup():
    import oracle as O
    from paper_2511_13386_b200 import configs

    c = configs.cfg2()
    grid = O.make_grid(256, 64)
    cfg = O.PConfig(eps=1e-2, t_final=0.5, ng=16, k_max=5, tol=1e-10,
                    opts=O.HOpts(adaptation=False))
    E0 = O.field(c.rho, c.rho_bar, grid)
    dt_c, dt_f = O.default_steps(cfg, grid, E0)
    return O, c, grid, cfg, dt_c, dt_f


def _cpu_cfg2_jump(args):
    """The reference's _jump_task (parareal.py:193-203) for window n."""
    n, rho_in = args
    O, c, grid, cfg, dt_c, dt_f = _cpu_cfg2_setup()
    t0 = time.perf_counter()
    f_rho, _ = O.fine_window(n, rho_in, c.g.reshape(256, 64), cfg, dt_f, grid, c.rho_bar)
    t_fine = time.perf_counter() - t0
    return n, f_rho - O.coarse(rho_in, n, cfg, dt_c, grid, c.rho_bar), t_fine


class CpuPool:
    """Pre-started, pre-imported worker pool (spawn) over the host cores."""

    def __init__(self, procs=None):
        import multiprocessing as mp

        self.procs = procs or min(os.cpu_count() or 1, 64)
        self.pool = mp.get_context("spawn").Pool(self.procs, initializer=_cpu_init)
        self.pool.map(_cpu_warm, range(4 * self.procs))

    def close(self):
        self.pool.close()
        self.pool.join()

    def cfg5(self, nsteps=100, n_inst=None):
        """Kinetic cell-updates/s of the oracle over all workers at once:
        total updates / (last stepping end - first stepping start).  Default
        sample: two instances per worker x 100 steps (~15 core-seconds)."""
        n_inst = n_inst or 2 * self.procs
        spans = self.pool.map(_cpu_cfg5, [(s, nsteps) for s in range(n_inst)], chunksize=1)
        wall = max(b for _, b in spans) - min(a for a, _ in spans)
        per_core = statistics.median(b - a for a, b in spans)
        upd = n_inst * nsteps * NX * NV
        return {"value": upd / wall, "unit": UNIT, "cores": self.procs, "kind": "port",
                "per_core": nsteps * NX * NV / per_core,
                "sample": f"{n_inst} cfg5 instances x {nsteps} steps (1024x128) on {self.procs} "
                          f"worker processes (pool pre-started, instance built outside the "
                          f"timed stepping), stepping span {wall:.2f} s"}

    def cfg2_parareal(self):
        """BASELINE cfg2 through the oracle's parareal algorithm
        (parareal.py:210-353): coarse sweep, then per iteration the jumps of
        all active windows on the pool (the reference's ThreadPool, as
        processes), the sequential correction here.  Wall time of the whole
        run, and the fine core-seconds (= the 1-worker fine time)."""
        O, c, grid, cfg, dt_c, dt_f = _cpu_cfg2_setup()
        t0 = time.perf_counter()
        ng = cfg.ng
        row = np.empty((ng + 1, grid.nx))
        row[0] = c.rho
        rho, t = c.rho, 0.0
        for n in range(1, ng + 1):
            rho, _ = O.fluid_advance(rho, t, float(cfg.bounds[n]), dt_c, grid, c.rho_bar, None)
            t = float(cfg.bounds[n])
            row[n] = rho
        rows, errs, fine_cs = [row], [], 0.0
        status = "max_iterations"
        for k in range(cfg.k_max):
            rk = rows[k]
            res = self.pool.map(_cpu_cfg2_jump, [(n, rk[n - 1]) for n in range(k + 1, ng + 1)],
                                chunksize=1)
            deltas = {n: d for n, d, _ in res}
            fine_cs += sum(tf for _, _, tf in res)
            new = rk.copy()
            for n in range(k + 1, ng + 1):
                new[n] = O.coarse(new[n - 1], n, cfg, dt_c, grid, c.rho_bar) + deltas[n]
            err = float(np.max(np.abs(new - rk)))
            rows.append(new)
            errs.append(err)
            if err < cfg.tol:
                status = "converged"
                break
        wall = time.perf_counter() - t0
        return {"wall_s": wall, "iterations": len(errs), "status": status, "cores": self.procs,
                "fine_core_s": fine_cs, "kind": "port",
                "sample": "full run: oracle parareal, window jumps on a process pool"}, rows


def run_reference(args):
    """Reference arm: the CPU implementation of the path (the oracle port;
    the reference is pure Python and cannot travel to the box) on all host
    cores, same metric / unit / config as the B200 arm.  Rank 0 only."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    pool = CpuPool()
    per = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = pool.cfg5()
        if i >= args.warmup:
            per.append(cb["value"])
    v = statistics.median(per)
    par, _ = pool.cfg2_parareal()
    pool.close()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(ws),
            "cpu_baseline": {**cb, "value": v},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "parareal": {"config": "cfg2: Nx=256, Nv=64, eps=1e-2, T=0.5, 16 slices, "
                                   "reference dt", **par}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------


def relaunch(n):
    """--gpus N > 1 outside torchrun: one rank per GPU on this node."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    ws, rank, local = dist_env()
    if ws != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; measuring {ws} rank(s)",
              file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)

    import torch

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
    del pipe, ens

    extra = {}
    if not args.no_extras:
        # collectives: every rank runs the engine (windows dealt across ranks)
        def guarded(fn, *a, **kw):
            # an extra that fails (on every rank alike) is reported, not fatal:
            # the headline line must still print
            try:
                return fn(*a, **kw)
            except Exception as ex:  # noqa: BLE001
                return {"error": f"{type(ex).__name__}: {ex}"[:400]}

        par = guarded(parareal_cfg2, barrier, maxr, peak)
        gpu_rows = par.pop("_rows", None)
        c4 = guarded(cfg4_sample, barrier, maxr, peak, ws)
        c3 = guarded(cfg3_iteration1, barrier, peak)   # run() is collective: every rank
        c5f = guarded(cfg5_fast, ens_args=(m, eps, dts, rb, rho_d, g_d, upd_rank),
                      barrier=barrier, maxr=maxr, peak=peak, ws=ws)
        barrier()
        if rank == 0:
            extra["parareal"] = par
            extra["cfg4"] = c4
            extra["cfg3"] = c3
            extra["cfg5_fast_mode"] = c5f
            extra["v3"] = guarded(v3_default_grid, peak)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "fine_kernel_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f)
        if tr.get("nv") == NV and tr.get("nx") == NX:
            traffic = tr.get("bytes_per_launch")
    cpu = None
    if rank == 0 and not args.no_cpu:
        pool = CpuPool()
        cpu = pool.cfg5()
        if "parareal" in extra and gpu_rows is not None:
            cpar, crows = pool.cfg2_parareal()
            cpar["gpu_ledger_bitwise_equal"] = bool(
                len(crows) == len(gpu_rows) and all(np.array_equal(a, b)
                                                    for a, b in zip(crows, gpu_rows)))
            extra["parareal"]["cpu"] = cpar
            extra["parareal"]["cpu_over_gpu_wall"] = cpar["wall_s"] / extra["parareal"]["wall_s"]
        pool.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(ws),
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
        barrier()      # rank 0's CPU baseline runs after the GPU work
        torch.distributed.destroy_process_group()


def _event():
    import torch

    return torch.cuda.Event(enable_timing=True)


def cfg5_fast(ens_args, barrier, maxr, peak, ws, reps=3):
    """The headline workload in fast scan mode (pk.scan_mode(False): the field
    solves' prefix sums parallel, not bitwise -- within 1e-10 relative L2 of
    the reference, tests/test_fast_mode.py).  Device-resident, CUDA events
    around `reps` 500-step launches, max over ranks."""
    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200.ensemble import Ensemble

    m, eps, dts, rb, rho_d, g_d, upd_rank = ens_args
    with pk.scan_mode(False):
        ens = Ensemble(m, eps, dts, rb)
        ens.load(rho_d, g_d)
        ens.run(NSTEPS)
        barrier()
        e0, e1 = _event(), _event()
        e0.record()
        for _ in range(reps):
            ens.load(rho_d, g_d)
            ens.run(NSTEPS, check=False)
        e1.record()
        barrier()
        ens.dev.check()
    ms = maxr(e0.elapsed_time(e1)) / reps
    val = upd_rank * ws / (ms * 1e-3)
    return {"value": val, "unit": UNIT, "ms_per_step": ms,
            "roofline_frac": val * BYTES_PER_UPDATE / (peak * 1e9),
            "mode": "fast scan (not bitwise; 1e-10 relative L2 bar)"}


def parareal_cfg2(barrier, maxr, peak):
    """BASELINE configs[1] through the drop-in run() on every rank (the engine
    deals the windows of each iteration across ranks and all-gathers the fine
    results).  Wall time = CUDA-event span on each rank's device timeline
    (host gaps between launches included), max over ranks."""
    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs

    c = configs.cfg2()
    cfg = pk.PararealConfig(eps=1e-2, t_final=0.5, ng=16, k_max=5, tol=1e-10,
                            options=pk.HybridOptions(adaptation=False))
    out = {"config": "cfg2: Nx=256, Nv=64, eps=1e-2, T=0.5, 16 slices, reference dt"}
    rows = None
    for mode, exact in (("exact", True), ("fast", False)):
        with pk.scan_mode(exact):
            pk.run(cfg, c.rho, c.g, c.mesh, c.rho_bar)  # warm-up
            barrier()
            e0, e1 = _event(), _event()
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
        r = {"wall_s": wall, "iterations": res.iterations, "status": res.status,
             "fine_s": maxr(tm.fine_total), "correction_s": maxr(tm.correction_total),
             "coarse_sweep_s": maxr(tm.coarse_sweep), "fine_cell_updates": fine_updates,
             # the whole parareal wall as a fraction of the HBM roofline at
             # 16 B per fine cell-update (latency-bound: 16 windows of 128 KiB)
             "hbm_frac_of_wall": fine_updates * BYTES_PER_UPDATE / wall / (peak * 1e9)}
        if exact:
            out.update(r)
            rows = [np.asarray(x) for x in res.ledger.rho]
        else:
            out["fast_mode"] = r
    out["_rows"] = rows
    return out


def cfg3_iteration1(barrier, peak):
    """BASELINE configs[2] (Nx=512, Nv=128, eps(x), thresholds 1e-3, 32 slices)
    on this GPU.  (a) The fine sweep of parareal iteration 1 -- all 32 windows
    from the coarse sweep's rows, one launch of the hybrid fine kernel, with
    the field guard relaxed to 1e-2 (the reference guard trips in window 2 at
    step 377) -- CUDA events around the launch, the kinetic rows
    the kernel streamed counted on the device (pk_count_rows): hybrid
    algorithmic bytes = 16 B x nv x kinetic rows + 8 B x nv x zeroed rows.
    (b) The drop-in run() end to end under both guards (wall until the typed
    error the reference raises too; tests/test_cfg3_parity.py pins where)."""
    import torch

    import paper_2511_13386_b200 as pk
    import paper_2511_13386_b200.parareal as ppl
    from paper_2511_13386_b200 import configs

    c = configs.cfg3()
    m = c.mesh
    cfg = pk.PararealConfig(eps=c.eps, t_final=1.0, ng=32, k_max=50, tol=1e-8,
                            thresholds=pk.Thresholds(1e-3, 1e-3),
                            options=pk.HybridOptions(adaptation=True))
    E0 = pk.solve_field(c.rho, c.rho_bar, m)
    fluid_p, kin_p = ppl.default_params(cfg, m, E0)
    nf, rem = pk.fluid.substep_sizes(0.0, 1.0 / 32, kin_p.dt)
    steps = nf + (1 if rem > 0.0 else 0)
    out = {"config": "cfg3: Nx=512, Nv=128, eps(x)=1e-3+0.5exp(-20(x-pi)^2), delta0=eta0=1e-3, "
                     "32 slices, T=1, reference dt", "fine_steps_per_window": steps}
    old = ppl.ADAPTIVE_FIELD_RTOL
    try:
        for mode, exact in (("exact", True), ("fast", False)):
            r = {}
            with pk.scan_mode(exact):
                ppl.ADAPTIVE_FIELD_RTOL = 1e-2
                eng = ppl._Engine(cfg, m, c.rho, c.g, c.rho_bar, fluid_p, kin_p)
                eng.coarse_sweep()
                X = eng.row[0:32].clone()
                dev = eng.be.dev
                cnt = torch.zeros((32, 2), dtype=torch.int64, device=X.device)
                eng.be.fine(X, list(range(1, 33)))        # warm-up
                torch.cuda.synchronize()
                dev.count_rows(cnt)
                e0, e1 = _event(), _event()
                e0.record()
                F, kc = eng.be.fine(X, list(range(1, 33)))
                e1.record()
                torch.cuda.synchronize()
                dev.count_rows(None)
                fine_s = e0.elapsed_time(e1) * 1e-3
                rows, zrows = (int(v) for v in cnt.sum(dim=0).tolist())
                alg = 16 * m.nv * rows + 8 * m.nv * zrows
                r.update({"iter1_fine_s": fine_s, "iter1_fine_us_per_step": fine_s / steps * 1e6,
                          "nominal_cell_updates": 32 * steps * m.nx * m.nv,
                          "kinetic_rows_streamed": rows, "rows_zeroed": zrows,
                          "kinetic_fraction_of_updates": rows / (32 * steps * m.nx),
                          "kinetic_cell_updates_per_s": rows * m.nv / fine_s,
                          "hbm_achieved_gbs": alg / fine_s / 1e9,
                          "hbm_frac": alg / fine_s / (peak * 1e9)})
                for guard, rt in (("reference_guard", old), ("relaxed_guard_1e-2", 1e-2)):
                    ppl.ADAPTIVE_FIELD_RTOL = rt
                    barrier()
                    t0 = time.perf_counter()
                    try:
                        res = pk.run(cfg, c.rho, c.g, m, c.rho_bar)
                        st = f"{res.status} after {res.iterations} iterations"
                    except pk.SimulationError as ex:
                        st = f"raised {type(ex).__name__} ({ex})"
                    torch.cuda.synchronize()
                    r[guard] = {"outcome": st, "wall_s": time.perf_counter() - t0}
            out["exact" if exact else "fast_mode"] = r
    finally:
        ppl.ADAPTIVE_FIELD_RTOL = old
    return out


def cfg4_sample(barrier, maxr, peak, ws, fine_steps=100):
    """BASELINE configs[3] (Nx=8192, Nv=256, v*=10, eps(x), 64 slices): one
    parareal iteration at a reduced T (every window = `fine_steps` fine steps
    at the reference dt; the full T = 2 needs 452,550 per window) through the
    drop-in run() on all ranks, reference guard.  Wall max over ranks; per
    fine step and per coarse step times, and the full-T extrapolation."""
    import torch

    import paper_2511_13386_b200 as pk
    import paper_2511_13386_b200.parareal as ppl
    from paper_2511_13386_b200 import configs

    c = configs.cfg4()
    m = c.mesh
    th = pk.Thresholds(1e-3, 1e-3)
    ng = 64
    cfg_full = pk.PararealConfig(eps=c.eps, t_final=2.0, ng=ng, k_max=1, tol=1e-8,
                                 thresholds=th, options=pk.HybridOptions(adaptation=True))
    E0 = pk.solve_field(c.rho, c.rho_bar, m, rtol=ppl.ADAPTIVE_FIELD_RTOL)
    fluid_p, kin_p = ppl.default_params(cfg_full, m, E0)
    nf_full, rem_full = pk.fluid.substep_sizes(0.0, 2.0 / ng, kin_p.dt)
    cf_full, crem_full = pk.fluid.substep_sizes(0.0, 2.0 / ng, fluid_p.dt)
    t_red = ng * fine_steps * kin_p.dt
    cfg = pk.PararealConfig(eps=c.eps, t_final=t_red, ng=ng, k_max=1, tol=1e-8, thresholds=th,
                            options=pk.HybridOptions(adaptation=True))
    cnf, crem = pk.fluid.substep_sizes(0.0, t_red / ng, fluid_p.dt)
    csteps = cnf + (1 if crem > 0.0 else 0)
    full_steps = nf_full + (1 if rem_full > 0.0 else 0)
    full_csteps = cf_full + (1 if crem_full > 0.0 else 0)
    out = {"config": f"cfg4: Nx=8192, Nv=256, v*=10, eps(x) as cfg3, 64 slices "
                     f"({-(-ng // ws)} per GPU on {ws}), delta0=eta0=1e-3; ONE iteration at a "
                     f"reduced T ({fine_steps} fine steps per window), reference guard",
           "fine_steps_per_window": fine_steps, "coarse_steps_per_window": csteps,
           "full_T_fine_steps_per_window": full_steps,
           "full_T_coarse_steps_per_window": full_csteps}
    for exact in (True, False):
        r = {}
        with pk.scan_mode(exact):
            try:
                pk.run(cfg, c.rho, c.g, m, c.rho_bar)    # warm-up
                barrier()
                e0, e1 = _event(), _event()
                e0.record()
                res = pk.run(cfg, c.rho, c.g, m, c.rho_bar)
                e1.record()
                barrier()
                tm = res.ledger.timings
                wall = maxr(e0.elapsed_time(e1) * 1e-3)
                fine_s = maxr(tm.fine_total)
                r.update({"status": res.status, "wall_s": wall, "fine_s": fine_s,
                          "coarse_sweep_s": maxr(tm.coarse_sweep),
                          "correction_s": maxr(tm.correction_total),
                          "kinetic_fraction_mean": float(np.mean(res.kinetic_fraction[1:]))})
                # F alone for one GPU's share at 8 GPUs: 8 lifted windows, one
                # launch of `fine_steps` steps, kinetic rows counted on the device
                eng = ppl._Engine(cfg, m, c.rho, c.g, c.rho_bar, fluid_p, kin_p)
                eng.coarse_sweep()
                X = eng.row[1:9].clone()
                cnt = torch.zeros((8, 2), dtype=torch.int64, device=X.device)
                eng.be.fine(X, list(range(2, 10)))       # warm-up
                torch.cuda.synchronize()
                eng.be.dev.count_rows(cnt)
                e4, e5 = _event(), _event()
                e4.record()
                eng.be.fine(X, list(range(2, 10)))
                e5.record()
                torch.cuda.synchronize()
                eng.be.dev.count_rows(None)
                f8 = e4.elapsed_time(e5) * 1e-3
                rows, zrows = (int(v) for v in cnt.sum(dim=0).tolist())
                alg = 16 * m.nv * rows + 8 * m.nv * zrows
                r.update({"fine_us_per_step_8_windows": f8 / fine_steps * 1e6,
                          "kinetic_fraction_of_updates_8_windows": rows / (8 * fine_steps * m.nx),
                          "hbm_frac_8_windows": alg / f8 / (peak * 1e9)})
                # G alone: one coarse chain of `csteps` steps per window on one GPU
                dev = pk.engine.Device.for_mesh(m)
                rho_d = dev.t(np.ascontiguousarray(c.rho.reshape(1, -1)))
                outb = dev.t(np.zeros((1, 8, m.nx)))
                rbd = dev.t(np.array([float(c.rho_bar)]))
                nfull = np.full((1, 8), 500, dtype=np.int32)
                for _ in range(2):
                    e2, e3 = _event(), _event()
                    e2.record()
                    dev.chain(rho_d, outb, None, None, None, nfull, np.zeros((1, 8)),
                              fluid_p.dt, rbd, ppl.ADAPTIVE_FIELD_RTOL, m2=fluid_p.m2)
                    e3.record()
                    torch.cuda.synchronize()
                dev.check()
                coarse_step = e2.elapsed_time(e3) * 1e-3 / (8 * 500)
                fine_step = fine_s / fine_steps
                r.update({"coarse_us_per_step": coarse_step * 1e6,
                          "fine_us_per_step_all_local_windows": fine_step * 1e6,
                          "extrapolated_full_T_coarse_sweep_s": coarse_step * full_csteps * ng,
                          # one iteration at full T on 8 GPUs, phase by phase:
                          # 8 windows of F per GPU, then the 64-window correction
                          "extrapolated_full_T_iteration_s_8gpu_phase_by_phase":
                              f8 / fine_steps * full_steps + coarse_step * full_csteps * ng})
            except pk.SimulationError as ex:
                r["status"] = f"raised {type(ex).__name__} ({ex})"
        out["exact" if exact else "fast_mode"] = r
    return out


def v3_default_grid(peak, nx=128, B=37, steps=20):
    """The reference's own 1D-3V default velocity grid (32 x 16 x 16 nodes per
    interface), B seeded-recipe instances of nx cells through the ensemble API,
    all-kinetic steps at the reference stable dt: device-resident fine
    throughput (CUDA events around one launch of `steps` steps, after a
    warm-up launch) and its fraction of the HBM roofline at 16 B per update."""
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
        e0, e1 = _event(), _event()
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
            "layout": {2: f"one CTA per row, clusters of {C}", 3: f"one CTA per row, software groups of {C}"}.get(layout, "warp per row")}


if __name__ == "__main__":
    main()
