"""Parallel-in-time driver (parareal.py:1-452), device-resident.

Algorithm 1 of the paper with the reference's semantics: coarse sweep, jumps
Delta^n = F(rho^{n-1,k}) - G(rho^{n-1,k}) for the unconverged windows
n = k+1..Ng, sequential correction rho^{n,k+1} = G(rho^{n-1,k+1}) + Delta^n,
successive error max|row_{k+1} - row_k|, stop at err < tol or k_max.

B200 design:
  * all active windows of an iteration are ONE launch of the persistent fine
    kernel (one thread-block cluster per window, libpk pk_fine_propagate);
  * G(rho^{n-1,k}) is taken from the previous correction / the coarse sweep
    instead of being recomputed (bit-identical);
  * the correction and the coarse sweep are one launch each (one CTA walks the
    windows sequentially with rho/E in shared memory, pk_coarse_chain);
  * multi-GPU: one process per GPU (torch.distributed, NCCL); the active
    windows are dealt cyclically to ranks, the fine results are all-gathered
    (the only exchange, (Ng - k) x nx doubles per iteration), and every rank
    runs the cheap correction redundantly, so the ledgers are bit-identical on
    all ranks and no broadcast is needed.  Results do not depend on the
    number of GPUs (cf. tests/test_parareal.py:93-101).
The host only forms schedules and reads one scalar (err) per iteration.

``_fine_window`` keeps the reference's plugin seam (parareal.py:153-190): if
it is monkeypatched, ``parareal_iterate`` calls it per window exactly as the
reference's ``_jump_task`` does.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .adaptation import Thresholds
from . import _native
from .engine import Device, make_phase
from .errors import NonFiniteState, SimulationError, code_of, raise_for
from .fluid import FluidStepParams, fluid_propagate, substep_sizes
from .hybrid import HybridOptions, HybridState, hybrid_propagate, knobs_of
from .kinetic import KineticStepParams
from .lifting import lift
from .mesh import MacroState, MicroState, PhaseMesh
from .poisson import SOLVABILITY_RTOL, solve_field

WORKERS_ENV = "PARAKIN_WORKERS"
_BACKEND = None   # engine backend factory; None = DeviceBackend (tests inject a CPU one)
ADAPTIVE_FIELD_RTOL = 1e-5


def field_guard(cfg: "PararealConfig"):
    return ADAPTIVE_FIELD_RTOL if cfg.options.adaptation else None


@dataclass(frozen=True)
class PararealConfig:
    eps: object
    t_final: float
    ng: int
    k_max: int = 50
    tol: float = 1e-10
    workers: int = 1
    parareal_enabled: bool = True
    thresholds: Thresholds = Thresholds(1e-5, 1e-5)
    options: HybridOptions = HybridOptions()

    def __post_init__(self):
        if self.ng < 1:
            raise ValueError("ng must be >= 1")
        if self.tol <= 0.0:
            raise ValueError("tol must be positive")

    @property
    def boundaries(self) -> np.ndarray:
        return np.linspace(0.0, self.t_final, self.ng + 1)


@dataclass
class PhaseTimings:
    coarse_sweep: float = 0.0
    fine_max: float = 0.0
    fine_total: float = 0.0
    lift_max: float = 0.0
    lift_total: float = 0.0
    fluid_window_max: float = 0.0
    correction_total: float = 0.0
    wall_total: float = 0.0
    iterations: list = field(default_factory=list)


@dataclass
class PararealLedger:
    boundaries: np.ndarray
    rho: list
    jumps: list = field(default_factory=list)
    err: list = field(default_factory=list)
    kinetic_fraction: np.ndarray | None = None
    timings: PhaseTimings = field(default_factory=PhaseTimings)

    def masses(self, dx: float) -> np.ndarray:
        return np.stack([row.sum(axis=1) * dx for row in self.rho])


@dataclass
class RunResult:
    status: str
    iterations: int
    ledger: PararealLedger
    boundary_rho: np.ndarray
    kinetic_fraction: np.ndarray
    config: PararealConfig

    def boundary_fields(self, mesh: PhaseMesh, rho_bar: float) -> np.ndarray:
        rtol = field_guard(self.config)
        return np.stack([solve_field(r, rho_bar, mesh, rtol=rtol) for r in self.boundary_rho])


def resolve_workers(requested: int | None = None) -> int:
    env = os.environ.get(WORKERS_ENV)
    if env:
        return max(1, int(env))
    if requested is not None and requested > 0:
        return requested
    return 1


def default_params(cfg: PararealConfig, mesh: PhaseMesh, E0) -> tuple:
    """parareal.py:138-146."""
    fluid_p = FluidStepParams.default(mesh)
    kin_p = KineticStepParams.default(mesh, cfg.eps, e_max=float(np.max(np.abs(E0))))
    return fluid_p, kin_p


# ---------------------------------------------------------------------------
# communicator (one process per GPU)


class _Comm:
    def __init__(self):
        self.rank, self.size, self.dist = 0, 1, None
        try:
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized():
                self.dist = dist
                self.rank, self.size = dist.get_rank(), dist.get_world_size()
        except Exception:
            pass

    def broadcast(self, t, src):
        """Broadcast t from rank src, stream-ordered on the current stream:
        NCCL returns a work whose wait() makes the current stream wait; a
        host-side backend (gloo) is staged through host memory (blocking)."""
        if self.size == 1:
            return None
        if t.is_cuda and self.dist.get_backend() != "nccl":
            h = t.detach().cpu()
            self.dist.broadcast(h, src)
            t.copy_(h)
            return None
        return self.dist.broadcast(t, src, async_op=True)

    def all_gather(self, t):
        """NCCL gathers device tensors directly (NVLink); a host-side backend
        (gloo: CPU test runs, or several ranks sharing one GPU) is staged
        through host memory."""
        if self.size == 1:
            return [t]
        import torch
        if t.is_cuda and self.dist.get_backend() != "nccl":
            parts = [torch.empty(t.shape, dtype=t.dtype) for _ in range(self.size)]
            self.dist.all_gather(parts, t.detach().cpu().contiguous())
            return [p.to(t.device) for p in parts]
        parts = [torch.empty_like(t) for _ in range(self.size)]
        self.dist.all_gather(parts, t.contiguous())
        return parts


# ---------------------------------------------------------------------------
# engine: coordination logic over a backend of five primitives


class DeviceBackend:
    """The product backend: libpk kernels on this rank's CUDA device.

    ``fine``   all listed windows in ONE persistent-kernel launch
               (pk_fine_propagate; window 1 from g0, others lifted);
    ``chain``  one CTA walks consecutive windows sequentially
               (pk_coarse_chain), optionally adding the jumps;
    ``many``   independent single-window G chains (cold G cache);
    ``jump`` / ``maxdiff``  Delta = F - G and max|a - b| with the
               reference's non-finite checks (parareal.py:267-269,283-286).
    """

    def __init__(self, eng):
        import torch

        self.torch = torch
        self.eng = eng
        self.dev = Device.for_mesh(eng.mesh)
        self.device = self.dev.device
        self.rb1 = self.dev.t(np.array([eng.rho_bar]))
        self.g0 = self.dev.t(np.ascontiguousarray(np.asarray(eng.g0, float).reshape(eng.nx, eng.nv)))
        self.err_d = torch.zeros(1, dtype=torch.float64, device=self.device)
        self._prep = {}   # window schedule -> prepared phases (fine)

    def tensor(self, a):
        return self.dev.t(np.ascontiguousarray(a, dtype=float))

    def chain(self, x, n0, n1, delta, rtol):
        e = self.eng
        W = n1 - n0 + 1
        out = self.torch.empty((W, e.nx), dtype=self.torch.float64, device=self.device)
        gout = self.torch.empty_like(out)
        sc = e.sc[n0 - 1:n1]
        self.dev.chain(x.reshape(1, e.nx), out.reshape(1, W, e.nx), gout.reshape(1, W, e.nx), None,
                       None if delta is None else delta.contiguous().reshape(1, W, e.nx),
                       [q[0] for q in sc], [q[1] for q in sc], e.fluid_p.dt, self.rb1,
                       SOLVABILITY_RTOL if rtol is None else rtol, m2=e.fluid_p.m2)
        self.dev.check()
        return out, gout

    def many(self, X, windows, rtol):
        e = self.eng
        B = len(windows)
        out = self.torch.empty((B, 1, e.nx), dtype=self.torch.float64, device=self.device)
        sc = [e.sc[n - 1] for n in windows]
        self.dev.chain(X.contiguous(), out, None, None, None, [q[0] for q in sc],
                       [q[1] for q in sc], e.fluid_p.dt, self.rb1.expand(B).contiguous(),
                       SOLVABILITY_RTOL if rtol is None else rtol, m2=e.fluid_p.m2)
        self.dev.check()
        return out[:, 0]

    def fine(self, X, windows):
        torch, dev, e = self.torch, self.dev, self.eng
        B = len(windows)
        nx, nv = e.nx, e.nv
        rho = X.clone()
        g = dev.scratch("par_g", (B, nx, nv))
        flags = []
        for i, n in enumerate(windows):
            if n == 1:
                g[i].copy_(self.g0)
                flags.append(2)      # true g0, E_prev := E  (parareal.py:169-170,178)
            else:
                flags.append(3)      # lifted g, E_prev := E
        E = torch.empty((B, nx), dtype=torch.float64, device=self.device)
        Ep = torch.empty_like(E)
        kc = torch.ones((B, nx), dtype=torch.uint8, device=self.device)
        ki = torch.ones_like(kc)
        eps = [e.cfg.eps] * B
        # phase coefficients (per-interface kappas for eps(x): host Python
        # floats, ~30 ms at nx = 8192) are built and uploaded once per window
        # schedule and reused by every iteration with the same one
        from . import engine as _engine

        key = (_engine.EXACT,) + tuple(e.sf[n - 1] for n in windows)
        prep = self._prep.get(key)
        if prep is None:
            dt = e.kin_p.dt
            ph0 = make_phase(e.mesh, eps, [dt] * B, [e.sf[n - 1][0] for n in windows])
            ph1 = make_phase(e.mesh, eps,
                             [e.sf[n - 1][1] if e.sf[n - 1][1] > 0.0 else dt for n in windows],
                             [1 if e.sf[n - 1][1] > 0.0 else 0 for n in windows])
            prep = self._prep[key] = ([ph0, ph1],
                                      dev.prepare_fine(B, [ph0, ph1], e.knobs, eps))
        dev.fine(rho, E, Ep, kc, ki, g, self.rb1.expand(B).contiguous(), flags, prep[0],
                 e.knobs, eps, e.rtol_f, prepared=prep[1])
        dev.check()   # the lowest failing slice (pk_device.cuh set_status)
        return rho, kc.sum(dim=1, dtype=torch.int64)

    def jump(self, F, G):
        delta = self.torch.empty_like(F)
        self.dev.jump(F, G, delta)
        self.dev.check()
        return delta

    def maxdiff(self, a, b):
        self.dev.maxdiff(a, b, self.err_d)
        err = float(self.err_d.item())
        self.dev.check()
        return err

    def clock(self):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record()
        return ev

    @staticmethod
    def seconds(a, b):
        return a.elapsed_time(b) * 1e-3


class _Engine:
    """State and coordination of one parareal run (parareal.py:210-310).

    Rows live on the backend's device; ``G[n]`` caches G(row_k[n-1]).  With
    a communicator of size > 1 the active windows are dealt cyclically to
    ranks, fine results are all-gathered, and every rank runs the
    (deterministic) correction itself, so ledgers agree bit for bit."""

    def __init__(self, cfg, mesh, rho0, g0, rho_bar, fluid_p, kin_p, comm=None, backend=None):
        import torch

        self.torch = torch
        self.cfg, self.mesh, self.fluid_p, self.kin_p = cfg, mesh, fluid_p, kin_p
        self.comm = comm or _Comm()
        self.rho_bar = float(rho_bar)
        self.g0 = g0
        self.nx, self.nv, ng = mesh.nx, mesh.nv, cfg.ng
        b = cfg.boundaries
        self.sc = [substep_sizes(float(b[n - 1]), float(b[n]), fluid_p.dt) for n in range(1, ng + 1)]
        self.sf = [substep_sizes(float(b[n - 1]), float(b[n]), kin_p.dt) for n in range(1, ng + 1)]
        for nf, rem in self.sc:
            if nf:
                fluid_p.check(fluid_p.dt, mesh)
            if rem > 0.0:
                fluid_p.check(rem, mesh)
        for nf, rem in self.sf:
            if nf:
                kin_p.check(kin_p.dt, mesh)
            if rem > 0.0:
                kin_p.check(rem, mesh)
        self.rtol = field_guard(cfg)
        self.rtol_f = SOLVABILITY_RTOL if self.rtol is None else self.rtol
        self.knobs = knobs_of(cfg.options, cfg.thresholds)
        self.be = backend(self) if backend is not None else DeviceBackend(self)
        self.row = self.be.tensor(np.repeat(np.asarray(rho0, float)[None], ng + 1, 0))
        self.G = torch.empty_like(self.row)
        self.overlap = None

    def close(self):
        """Wait for any speculative work still in flight (buffers stay owned
        until it has finished)."""
        if self.overlap is not None:
            self.overlap.sync()

    def coarse_sweep(self):
        """Row 0 (parareal.py:210-229); default field guard as the reference."""
        out, _ = self.be.chain(self.row[0], 1, self.cfg.ng, None, None)
        self.row[1:] = out
        self.G[1:] = out   # G(row_0[n-1]) == row_0[n]

    def cold_G(self, k):
        """G(row_k[n-1]) for n = k+1..Ng (independent chains)."""
        wins = list(range(k + 1, self.cfg.ng + 1))
        if wins:
            self.G[k + 1:] = self.be.many(self.row[k:self.cfg.ng], wins, self.rtol)

    def correct(self, k, delta):
        """The sequential correction of iteration k+1 as one chain launch
        (parareal.py:272-284); a field-guard failure is reported for the
        window it happened in (the chain stops there)."""
        try:
            return self.be.chain(self.row[k], k + 1, self.cfg.ng, delta, self.rtol)
        except SimulationError as ex:
            w = getattr(ex, "pk_step", None)
            if w is None or w < 0:
                raise
            raise_for(code_of(ex), f"correction, window {k + 1 + w}", None, None)

    def iterate(self, k):
        torch, cfg, be = self.torch, self.cfg, self.be
        ng, nx = cfg.ng, self.nx
        targets = list(range(k + 1, ng + 1))
        B = len(targets)
        if B == 0:
            # every window converged by prefix exactness: row_{k+1} == row_k
            return 0.0, self.row[:0], np.zeros(ng + 1), targets, 0.0, 0.0
        if use_overlap(self):
            if self.overlap is None:
                self.overlap = _Overlap.get(self)
            return self.overlap.iterate(k)
        t0 = be.clock()
        size, rank = self.comm.size, self.comm.rank
        if size == 1:
            Fall, kcount, fail = _fine_or_fail(be, self.row[k:ng], targets)
            if fail:
                raise_for(fail[0], f"window {fail[1]}, step {fail[2]}", fail[1], fail[2])
        else:
            # cyclic deal; one all-gather of [per + 2, nx] rows per rank (extra
            # rows: the kinetic-cell counts, and this rank's failure record)
            per = -(-B // size)
            assert per <= nx and nx >= 3, "window share exceeds the gather row width"
            mine = targets[rank::size]
            buf = torch.zeros((per + 2, nx), dtype=torch.float64, device=self.row.device)
            if mine:
                # never raise before the collective: the other ranks would
                # block in it forever.  Post (code, window, step) instead.
                Fr, kc, fail = _fine_or_fail(be, self.row[[n - 1 for n in mine]], mine)
                if fail:
                    buf[per + 1, :3] = torch.tensor(fail, dtype=torch.float64)
                else:
                    buf[:len(mine)] = Fr
                    buf[per, :len(mine)] = kc.to(torch.float64)
            parts = self.comm.all_gather(buf)
            fails = [tuple(int(v) for v in p[per + 1, :3].tolist()) for p in parts]
            fails = [f for f in fails if f[0] != 0]
            if fails:
                # every rank raises the lowest failing window's error, as the
                # reference consumes its window futures in order (parareal.py:260-266)
                code, win, st = min(fails, key=lambda f: f[1])
                raise_for(code, f"window {win}, step {st}", win, st)
            Fall = torch.empty((B, nx), dtype=torch.float64, device=self.row.device)
            kcount = torch.empty(B, dtype=torch.int64, device=self.row.device)
            for r, part in enumerate(parts):
                for j, n in enumerate(targets[r::size]):
                    Fall[n - k - 1] = part[j]
                    kcount[n - k - 1] = part[per, j].to(torch.int64)
        t1 = be.clock()
        try:
            delta = be.jump(Fall, self.G[k + 1:])   # NonFiniteState (parareal.py:267-269)
        except NonFiniteState:
            # name the lowest non-finite window, as the reference's message does
            bad = (~torch.isfinite(Fall - self.G[k + 1:])).any(dim=1).nonzero()
            n = targets[int(bad[0, 0])] if bad.numel() else targets[0]
            raise NonFiniteState(f"non-finite fine/coarse jump in window {n} (blow-up)") from None
        t2 = be.clock()
        new = self.row.clone()
        Gn = self.G.clone()
        out, gout = self.correct(k, delta)
        new[k + 1:] = out
        Gn[k + 1:] = gout
        t3 = be.clock()
        err = be.maxdiff(new, self.row)          # NonFiniteState (parareal.py:283-284)
        fracs = np.zeros(ng + 1)
        kc_h = kcount.cpu().numpy()
        for j, n in enumerate(targets):
            fracs[n] = float(kc_h[j]) / nx
        self.row, self.G = new, Gn
        return err, delta, fracs, targets, be.seconds(t0, t1), be.seconds(t2, t3)


def _fine_or_fail(be, X, windows):
    """be.fine over `windows`; a failure is returned as (code, window, step)
    of the lowest failing window instead of raised (the batch reports its
    lowest failing slice: pk_device.cuh set_status)."""
    try:
        F, kc = be.fine(X, windows)
        return F, kc, None
    except (SimulationError, ValueError) as ex:
        sl = getattr(ex, "pk_slice", None)
        win = windows[sl] if sl is not None and 0 <= sl < len(windows) else windows[0]
        st = getattr(ex, "pk_step", None)
        return None, None, (code_of(ex), win, -1 if st is None else int(st))


# Overlap the coarse correction with the next iteration's fine windows on a
# single GPU (tests can switch it off to compare the two schedules).
OVERLAP = True
TIMELINE = False    # diagnostics: record per-window event times (tools/par_timing.py)
OVERLAP_CACHE = 2   # schedules (with their contexts and buffers) kept for reuse


def use_overlap(eng) -> bool:
    """The overlapped schedule (below) when this rank's windows fit beside the
    correction: at most 32 (one stream each) and a small total footprint --
    otherwise persistent fine windows fill every SM and the correction's
    chain kernel waits behind whole windows (cfg4 on one GPU: 64 windows of
    8192 x 256 run phase by phase; on 8 GPUs, 8 per rank, overlapped)."""
    if not OVERLAP or not isinstance(eng.be, DeviceBackend):
        return False
    local = -(-eng.cfg.ng // eng.comm.size)
    return local <= 32 and local * eng.nx <= 65536


class _Overlap:
    """Parareal schedule with the coarse correction overlapped with the fine
    windows of the next iteration, on one GPU or one
    process per GPU.

    F for window n of iteration k+1 needs only row_{k+1}[n-1], which the
    correction of iteration k produces window by window.  So each window's F
    is enqueued, speculatively, behind the correction step that produces its
    input -- on the window's own stream and solver context (two per window,
    one per iteration parity, so workspaces and status records never mix) --
    and its jump behind the step that produces G(row_{k+1}[n-1]).  The
    correction runs window by window on its own stream.  Every window's jump
    travels as a payload [Delta (nx) | status code, step | kinetic cells]:
    the status record is stored on the device behind the jump
    (pk_status_store), so no host synchronisation sits in the pipeline.

    Several ranks: window n of iteration k belongs to rank (n - k - 1) % size
    (the phase-by-phase deal).  Every rank runs the whole correction itself
    (deterministic, so all ranks hold the same rows); before correction step
    n the owner broadcasts window n's payload (NCCL on the correction stream,
    behind the jump's event), so the correction -- and with it the next
    iteration's windows on every rank -- advances window by window as the
    jumps arrive instead of after a whole-iteration all-gather.  Failures
    travel in the payloads: every rank completes the same collectives and
    then raises the same error (lowest failing window first, fine before
    correction, as the reference's order, parareal.py:260-284).

    Events order all of it; the host reads err and the payloads from the
    correction stream.  Every value is the same function of the same inputs
    as in the phase-by-phase schedule, so ledgers are bitwise identical; the
    speculative work of an iteration that never happens is dropped unread."""

    _cache: dict = {}   # insertion-ordered: least recently used first

    @classmethod
    def get(cls, eng):
        """Resources are cached per (mesh, device, schedule, parameters): a
        repeated run reuses the solver contexts, prepared phases, buffers and
        streams.  At most OVERLAP_CACHE schedules are kept; an evicted one is
        synchronised before its contexts and buffers are released."""
        cfg = eng.cfg
        from . import engine as _eng

        key = (_eng.EXACT, id(eng.mesh), str(eng.be.device), cfg.ng, id(cfg.eps), eng.kin_p.dt,
               eng.fluid_p.dt, eng.fluid_p.m2, eng.rtol_f, repr(eng.knobs), tuple(eng.sf),
               tuple(eng.sc), eng.comm.size, eng.comm.rank)
        ov = cls._cache.pop(key, None)
        if ov is None or ov.mesh is not eng.mesh or ov.eps is not cfg.eps:
            ov = cls(eng)
        cls._cache[key] = ov
        while len(cls._cache) > max(1, OVERLAP_CACHE):
            old = cls._cache.pop(next(iter(cls._cache)))
            old.sync()
        ov.sync()
        ov.clear_status()
        ov.eng = eng
        ov.comm = eng.comm
        ov.Rn = eng.torch.empty_like(eng.row)
        ov.Gn = eng.torch.empty_like(eng.G)
        return ov

    def __init__(self, eng):
        torch = eng.torch
        self.torch, self.eng, self.comm = torch, eng, eng.comm
        self.mesh, self.eps = eng.mesh, eng.cfg.eps  # keep the key objects alive
        cfg, mesh, be = eng.cfg, eng.mesh, eng.be
        ng, nx, nv = cfg.ng, eng.nx, eng.nv
        dv = be.device
        # two solver contexts per window (one per iteration parity) + the correction's
        self.devs = [None] + [[Device(mesh, dv), Device(mesh, dv)] for _ in range(ng)]
        self.cdev = Device(mesh, dv)
        # torch hands out streams from a pool of 32 per priority: the
        # correction (the critical path) takes a high-priority stream of its
        # own; each window one low-priority stream for both parities
        self.cs = torch.cuda.Stream(dv, priority=-1)
        self.side = None  # cancel requests (sync)
        ws = [torch.cuda.Stream(dv) for _ in range(ng)]
        self.fs = [None] + [[s, s] for s in ws]
        f64 = dict(dtype=torch.float64, device=dv)
        # jump payloads per parity: [Delta (nx) | status code, step | kinetic cells]
        self.D = torch.zeros((2, ng + 1, nx + 3), **f64)
        self.Rn = torch.empty_like(eng.row)                     # next rows
        self.Gn = torch.empty_like(eng.G)                       # next G cache
        self.buf = [None] + [[dict(rho=torch.empty((1, nx), **f64), E=torch.empty((1, nx), **f64),
                                   Ep=torch.empty((1, nx), **f64),
                                   kc=torch.ones((1, nx), dtype=torch.uint8, device=dv),
                                   ki=torch.ones((1, nx), dtype=torch.uint8, device=dv),
                                   g=torch.empty((1, nx, nv), **f64)) for _ in range(2)]
                             for _ in range(ng)]
        eps, dt = cfg.eps, eng.kin_p.dt
        self.prep = [None] * (ng + 1)
        self.flags = [None] * (ng + 1)
        self.sched = [None] * (ng + 1)
        phases = {}
        for n in range(1, ng + 1):
            nf, rem = eng.sf[n - 1]
            key = (nf, rem)
            if key not in phases:
                phases[key] = [make_phase(mesh, [eps], [dt], [nf]),
                               make_phase(mesh, [eps], [rem if rem > 0.0 else dt],
                                          [1 if rem > 0.0 else 0])]
            self.prep[n] = [self.devs[n][q].prepare_fine(1, phases[key], eng.knobs, [eps])
                            for q in range(2)]
            # window 1 starts from the true g0, the others from a lift (parareal.py:169-178)
            self.flags[n] = be.dev.t(np.array([2 if n == 1 else 3], dtype=np.uint8))
            self.sched[n] = self.cdev.chain_schedule([eng.sc[n - 1][0]], [eng.sc[n - 1][1]],
                                                     eng.fluid_p.dt, eng.fluid_p.m2)
        self.ev_row = [torch.cuda.Event(enable_timing=TIMELINE) for _ in range(ng + 1)]
        self.ev_fstart = [[torch.cuda.Event(enable_timing=True) for _ in range(ng + 1)]
                          for _ in range(2)]
        self.ev_jump = [[torch.cuda.Event(enable_timing=True) for _ in range(ng + 1)]
                        for _ in range(2)]
        self.spec = None    # the iteration whose fine windows are already enqueued

    def owner(self, n, k):
        """Rank that runs window n in iteration k (the phase-by-phase deal)."""
        return (n - k - 1) % self.comm.size

    def _fine(self, q, n, x_row, wait):
        """Enqueue F for window n (parity q) from x_row [nx] after `wait`."""
        torch, eng = self.torch, self.eng
        s, dev, b = self.fs[n][q], self.devs[n][q], self.buf[n][q]
        with torch.cuda.stream(s):
            if wait is not None:
                s.wait_event(wait)
            if TIMELINE:
                self.ev_fstart[q][n].record(s)
            b["rho"][0].copy_(x_row)
            if n == 1:
                b["g"][0].copy_(eng.be.g0)
            b["kc"].fill_(1)
            b["ki"].fill_(1)
            dev.fine(b["rho"], b["E"], b["Ep"], b["kc"], b["ki"], b["g"], eng.be.rb1,
                     self.flags[n], None, eng.knobs, [eng.cfg.eps], eng.rtol_f,
                     prepared=self.prep[n][q])
            self.D[q, n, eng.nx + 2] = b["kc"].sum(dtype=torch.float64)

    def _jump(self, q, n, G_row, wait):
        """Enqueue Delta = F - G for window n (parity q) after `wait`, then the
        window context's status into the payload (re-arming the record)."""
        torch, nx = self.torch, self.eng.nx
        s, dev = self.fs[n][q], self.devs[n][q]
        with torch.cuda.stream(s):
            if wait is not None:
                s.wait_event(wait)
            dev.jump(self.buf[n][q]["rho"][0], G_row, self.D[q, n, :nx])
            dev._rc(dev.lib.pk_status_store(dev.ctx, C.c_void_p(self.D[q, n, nx:].data_ptr()), 1,
                                            C.c_void_p(s.cuda_stream)), "pk_status_store")
            self.ev_jump[q][n].record(s)

    def iterate(self, k):
        torch, eng = self.torch, self.eng
        cfg, ng, nx = eng.cfg, eng.cfg.ng, eng.nx
        size, rank = self.comm.size, self.comm.rank
        q = k & 1
        self._t_iter = time.perf_counter()
        targets = list(range(k + 1, ng + 1))
        R, Gc, Rn, Gn = eng.row, eng.G, self.Rn, self.Gn
        start = torch.cuda.Event(enable_timing=True)
        start.record(torch.cuda.current_stream())
        if self.spec != k:   # nothing speculative for this iteration: launch its windows now
            for n in targets:
                if self.owner(n, k) == rank:
                    self._fine(q, n, R[n - 1], start)
                    self._jump(q, n, Gc[n], None)
        speculate = k + 1 < cfg.k_max and k + 2 <= ng
        cs, cdev = self.cs, self.cdev
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(cs):
            cs.wait_event(start)
            Rn.copy_(R)           # prefix rows 0..k are final (prefix exactness)
            Gn.copy_(Gc)
            c0.record(cs)
        for n in targets:
            with torch.cuda.stream(cs):
                own = self.owner(n, k)
                if own == rank:
                    cs.wait_event(self.ev_jump[q][n])
                if size > 1:
                    # window n's payload from its owner, in window order on every rank
                    work = self.comm.broadcast(self.D[q, n], own)
                    if work is not None:
                        work.wait()
                # row_{k+1}[n] = G(row_{k+1}[n-1]) + Delta_k[n]; gout = G(row_{k+1}[n-1])
                cdev.chain_raw(Rn[n - 1].view(1, nx), Rn[n].view(1, 1, nx), Gn[n].view(1, 1, nx),
                               None, self.D[q, n, :nx].view(1, 1, nx), self.sched[n],
                               eng.fluid_p.dt, eng.be.rb1,
                               SOLVABILITY_RTOL if eng.rtol is None else eng.rtol)
                self.ev_row[n].record(cs)
            if speculate:
                if n + 1 <= ng and self.owner(n + 1, k + 1) == rank:
                    self._fine(q ^ 1, n + 1, Rn[n], self.ev_row[n])
                if n >= k + 2 and self.owner(n, k + 1) == rank:
                    self._jump(q ^ 1, n, Gn[n], self.ev_row[n])
        with torch.cuda.stream(cs):
            c1.record(cs)
            cdev.maxdiff(Rn, R, eng.be.err_d)
            self.host_enqueue_s = time.perf_counter() - self._t_iter
            err = float(eng.be.err_d.item())     # waits for the correction stream only
            pay = self.D[q, k + 1:, nx:].cpu().numpy()   # ordered behind every payload
        self.spec = k + 1 if speculate else None
        # the reference raises the fine windows' errors (lowest window first)
        # before any correction error (parareal.py:260-284)
        for j, n in enumerate(targets):
            if pay[j, 0] != 0.0:
                st = int(pay[j, 1])
                raise_for(int(pay[j, 0]), f"window {n}, step {st}", n, st)
        try:
            cdev.check_stream(cs)
        except SimulationError:
            # one window per launch here: locate the failing window with the
            # phase-by-phase correction (one launch; it raises for that window)
            self.sync()
            eng.correct(k, self.D[q, k + 1:, :nx])
            raise
        delta = self.D[q, k + 1:, :nx].clone()
        fracs = np.zeros(ng + 1)
        for j, n in enumerate(targets):
            fracs[n] = float(pay[j, 2]) / nx
        # fine span seen from this iteration's start (speculative windows may
        # have finished during the previous correction: then ~0); own windows
        mine = [n for n in targets if self.owner(n, k) == rank]
        t_fine = max([0.0] + [start.elapsed_time(self.ev_jump[q][n]) * 1e-3 for n in mine])
        t_corr = c0.elapsed_time(c1) * 1e-3
        if TIMELINE:
            self.timeline = [(n, start.elapsed_time(self.ev_fstart[q][n]),
                              start.elapsed_time(self.ev_jump[q][n]),
                              start.elapsed_time(self.ev_row[n])) for n in mine]
        # swap the row / G buffers: the speculative windows read the new ones
        eng.row, self.Rn = Rn, R
        eng.G, self.Gn = Gn, Gc
        return err, delta, fracs, targets, t_fine, t_corr

    def sweep(self):
        """Coarse sweep window by window (parareal.py:210-229; the reference's
        default field guard), the first iteration's windows (this rank's)
        enqueued behind the rows they start from, their jumps behind
        G(row_0[n-1]) == row_0[n]."""
        torch, eng = self.torch, self.eng
        ng, nx = eng.cfg.ng, eng.nx
        R, Gc, cs = eng.row, eng.G, self.cs
        t_host = time.perf_counter()
        start = torch.cuda.Event(enable_timing=TIMELINE)
        start.record(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            cs.wait_event(start)
        for n in range(1, ng + 1):
            with torch.cuda.stream(cs):
                self.cdev.chain_raw(R[n - 1].view(1, nx), R[n].view(1, 1, nx), Gc[n].view(1, 1, nx),
                                    None, None, self.sched[n], eng.fluid_p.dt, eng.be.rb1,
                                    SOLVABILITY_RTOL)
                self.ev_row[n].record(cs)
            if eng.cfg.k_max > 0 and self.owner(n, 0) == self.comm.rank:
                self._fine(0, n, R[n - 1], start if n == 1 else self.ev_row[n - 1])
                self._jump(0, n, Gc[n], self.ev_row[n])
        self.spec = 0 if eng.cfg.k_max > 0 else None
        self.sweep_enqueue_s = time.perf_counter() - t_host
        self.cdev.check_stream(cs)
        if TIMELINE:
            mine = [n for n in range(1, ng + 1) if self.owner(n, 0) == self.comm.rank]
            self.sweep_timeline = [(n, start.elapsed_time(self.ev_fstart[0][n]),
                                    start.elapsed_time(self.ev_row[n])) for n in mine]
            self.sweep_wait_s = time.perf_counter() - t_host

    def clear_status(self):
        """Drop status records latched by speculative work that was never
        consumed (an iteration that did not happen), before the contexts are
        reused by another run."""
        st = _native.PkStatus()
        for d in [self.cdev] + [d for pair in self.devs[1:] for d in pair]:
            d._rc(d.lib.pk_status_read(d.ctx, C.byref(st), 1), "status")
        self.D.zero_()

    def sync(self):
        """Wait for the work in flight.  Fine windows enqueued speculatively for
        an iteration that will not happen (the run converged, hit k_max or
        failed) are asked to stop first: they would run their whole window
        (cfg2: ~8 ms of a ~50 ms run) only to be dropped."""
        if self.spec is not None:
            torch = self.torch
            if self.side is None:
                self.side = torch.cuda.Stream(self.cs.device)
            for pair in self.devs[1:]:
                for d in pair:
                    d.cancel(self.side)
            self.side.synchronize()
        for pair in self.fs[1:]:
            pair[0].synchronize()
        self.cs.synchronize()
        self.spec = None


_ENGINES: dict = {}


# ---------------------------------------------------------------------------
# reference-facing API


def _fine_window(n, rho_in, g0, cfg: PararealConfig, kin_p: KineticStepParams, mesh: PhaseMesh,
                 rho_bar, ws=None):
    """F for window n-1 -> n from a boundary density (parareal.py:153-190).
    The plugin seam: replaceable by monkeypatching this module attribute."""
    t0, t1 = float(cfg.boundaries[n - 1]), float(cfg.boundaries[n])
    rtol = field_guard(cfg)
    E = solve_field(rho_in, rho_bar, mesh, rtol=rtol)
    tic = time.perf_counter()
    micro = MicroState(g=g0) if n == 1 else lift(
        rho_in, E, cfg.eps, mesh, order=cfg.options.lift_order,
        time_elim=cfg.options.time_elim, rho_bar=rho_bar)
    t_lift = time.perf_counter() - tic
    state = HybridState.initial(MacroState(rho=np.asarray(rho_in, float), E=E, t=t0), micro, mesh)
    tic = time.perf_counter()
    out = hybrid_propagate(state, t1, kin_p, cfg.thresholds, cfg.options, mesh, rho_bar,
                           field_rtol=rtol)
    return out.macro.rho, {"lift_s": t_lift, "fine_s": time.perf_counter() - tic,
                           "kinetic_fraction": out.labels.kinetic_fraction}


_ORIG_FINE_WINDOW = _fine_window


def _jump_task(n, row_k, g0, cfg, fluid_p, kin_p, mesh, rho_bar):
    """parareal.py:193-203 (host seam path)."""
    rho_in = row_k[n - 1]
    fine_rho, diag = _fine_window(n, rho_in, g0, cfg, kin_p, mesh, rho_bar)
    tic = time.perf_counter()
    coarse = fluid_propagate(MacroState(rho=rho_in, E=np.zeros_like(rho_in),
                                        t=cfg.boundaries[n - 1]),
                             cfg.boundaries[n], fluid_p, mesh, rho_bar, field_rtol=field_guard(cfg))
    diag["fluid_s"] = time.perf_counter() - tic
    return n, fine_rho - coarse.rho, diag


def coarse_sweep(rho0, cfg: PararealConfig, fluid_p: FluidStepParams, mesh: PhaseMesh,
                 rho_bar: float, g0=None, kin_p=None) -> PararealLedger:
    """Row 0 from the coarse propagator (parareal.py:210-229), one launch."""
    tic = time.perf_counter()
    bounds = cfg.boundaries
    ledger = PararealLedger(boundaries=bounds, rho=[])
    if kin_p is None:
        kin_p = KineticStepParams(eps=cfg.eps, dt=fluid_p.dt)
    if g0 is None:
        g0 = np.zeros((mesh.nx,) + mesh.vgrid.shape)
    eng = _Engine(cfg, mesh, rho0, g0, rho_bar, fluid_p, kin_p, backend=_BACKEND)
    if use_overlap(eng):
        eng.overlap = _Overlap.get(eng)
        eng.overlap.sweep()     # also starts iteration 0's windows
    else:
        eng.coarse_sweep()
    _ENGINES[id(ledger)] = eng
    ledger.rho.append(eng.row.cpu().numpy())
    ledger.kinetic_fraction = np.zeros(cfg.ng + 1)
    ledger.timings.coarse_sweep = time.perf_counter() - tic
    return ledger


def parareal_iterate(ledger: PararealLedger, k: int, cfg: PararealConfig,
                     fluid_p: FluidStepParams, kin_p: KineticStepParams, mesh: PhaseMesh,
                     rho_bar: float, g0, pool=None) -> float:
    """Consume row k, append row k+1; returns the successive error
    (parareal.py:232-310)."""
    iter_tic = time.perf_counter()
    tm = ledger.timings
    if _fine_window is not _ORIG_FINE_WINDOW:
        return _iterate_host_seam(ledger, k, cfg, fluid_p, kin_p, mesh, rho_bar, g0, iter_tic)
    eng = _ENGINES.get(id(ledger))
    if eng is None or eng.kin_p is not kin_p or k != len(ledger.rho) - 1:
        eng = _Engine(cfg, mesh, ledger.rho[0][0], g0, rho_bar, fluid_p, kin_p,
                      backend=_BACKEND)
        eng.row = eng.be.tensor(ledger.rho[k])
        eng.cold_G(k)   # G(row_k[n-1]) for the active windows
        _ENGINES[id(ledger)] = eng
    err, delta, fracs, targets, t_fine, t_corr = eng.iterate(k)
    ledger.rho.append(eng.row.cpu().numpy())
    dh = delta.cpu().numpy()
    ledger.jumps.append({n: dh[j] for j, n in enumerate(targets)})
    ledger.err.append(err)
    for n in targets:
        ledger.kinetic_fraction[n] = fracs[n]
    tm.fine_max = max(tm.fine_max, t_fine)
    tm.fine_total += t_fine
    tm.fluid_window_max = max(tm.fluid_window_max, t_corr / max(1, len(targets)))
    tm.correction_total += t_corr
    tm.iterations.append({"k": k + 1, "err": err, "parallel_s": t_fine, "correction_s": t_corr,
                          "wall_s": time.perf_counter() - iter_tic})
    return err


def _iterate_host_seam(ledger, k, cfg, fluid_p, kin_p, mesh, rho_bar, g0, iter_tic):
    """Reference-order iteration through a replaced ``_fine_window``."""
    row_k = ledger.rho[k]
    targets = range(k + 1, cfg.ng + 1)
    tic = time.perf_counter()
    deltas, diags = {}, {}
    for n in targets:
        _, deltas[n], diags[n] = _jump_task(n, row_k, g0, cfg, fluid_p, kin_p, mesh, rho_bar)
    for n in targets:
        if not np.isfinite(deltas[n]).all():
            raise NonFiniteState(f"non-finite fine/coarse jump in window {n} (blow-up)")
    t_par = time.perf_counter() - tic
    new_row = row_k.copy()
    tic = time.perf_counter()
    zero_E = np.zeros(mesh.nx)
    for n in targets:
        coarse = fluid_propagate(MacroState(rho=new_row[n - 1], E=zero_E, t=cfg.boundaries[n - 1]),
                                 cfg.boundaries[n], fluid_p, mesh, rho_bar,
                                 field_rtol=field_guard(cfg))
        new_row[n] = coarse.rho + deltas[n]
    t_corr = time.perf_counter() - tic
    if not np.isfinite(new_row).all():
        raise NonFiniteState(f"non-finite density after parareal iteration {k + 1}")
    err = float(np.max(np.abs(new_row - row_k)))
    ledger.rho.append(new_row)
    ledger.jumps.append(deltas)
    ledger.err.append(err)
    for n in targets:
        ledger.kinetic_fraction[n] = diags[n]["kinetic_fraction"]
    tm = ledger.timings
    tm.fine_max = max(tm.fine_max, max((d["fine_s"] for d in diags.values()), default=0.0))
    tm.fine_total += sum(d["fine_s"] for d in diags.values())
    tm.lift_max = max(tm.lift_max, max((d["lift_s"] for d in diags.values()), default=0.0))
    tm.lift_total += sum(d["lift_s"] for d in diags.values())
    tm.fluid_window_max = max(tm.fluid_window_max,
                              max((d["fluid_s"] for d in diags.values()), default=0.0))
    tm.correction_total += t_corr
    tm.iterations.append({"k": k + 1, "err": err, "parallel_s": t_par, "correction_s": t_corr,
                          "wall_s": time.perf_counter() - iter_tic})
    _ENGINES.pop(id(ledger), None)
    return err


def run(cfg: PararealConfig, rho0, g0, mesh: PhaseMesh, rho_bar: float) -> RunResult:
    """Coarse sweep then parareal iterations (parareal.py:313-353)."""
    wall_tic = time.perf_counter()
    E0 = solve_field(rho0, rho_bar, mesh)
    fluid_p, kin_p = default_params(cfg, mesh, E0)
    if not cfg.parareal_enabled:
        result = _serial_fine_run(cfg, rho0, g0, kin_p, mesh, rho_bar)
        result.ledger.timings.wall_total = time.perf_counter() - wall_tic
        return result
    ledger = coarse_sweep(rho0, cfg, fluid_p, mesh, rho_bar, g0=g0, kin_p=kin_p)
    status = "max_iterations"
    try:
        for k in range(cfg.k_max):
            err = parareal_iterate(ledger, k, cfg, fluid_p, kin_p, mesh, rho_bar, g0)
            if err < cfg.tol:
                status = "converged"
                break
    finally:
        eng = _ENGINES.pop(id(ledger), None)
        if eng is not None:
            eng.close()
    ledger.timings.wall_total = time.perf_counter() - wall_tic
    return RunResult(status=status, iterations=len(ledger.err), ledger=ledger,
                     boundary_rho=ledger.rho[-1], kinetic_fraction=ledger.kinetic_fraction,
                     config=cfg)


def _serial_fine_run(cfg, rho0, g0, kin_p, mesh, rho_bar) -> RunResult:
    """Serial fine baseline with state carried across windows (parareal.py:356-392)."""
    bounds = cfg.boundaries
    row = np.empty((cfg.ng + 1, mesh.nx))
    row[0] = rho0
    fractions = np.zeros(cfg.ng + 1)
    E0 = solve_field(rho0, rho_bar, mesh)
    state = HybridState.initial(MacroState(rho=rho0, E=E0, t=0.0), MicroState(g=g0), mesh)
    tic = time.perf_counter()
    for n in range(1, cfg.ng + 1):
        state = hybrid_propagate(state, bounds[n], kin_p, cfg.thresholds, cfg.options, mesh,
                                 rho_bar, field_rtol=field_guard(cfg))
        row[n] = state.macro.rho
        fractions[n] = state.labels.kinetic_fraction
    ledger = PararealLedger(boundaries=bounds, rho=[row])
    ledger.kinetic_fraction = fractions
    ledger.timings.fine_total = time.perf_counter() - tic
    return RunResult(status="serial", iterations=0, ledger=ledger, boundary_rho=row,
                     kinetic_fraction=fractions, config=cfg)


def lift_restart_reference(cfg, rho0, g0, mesh, rho_bar) -> np.ndarray:
    """The parareal fixed point: serial chain of lifted restarts (parareal.py:395-413)."""
    E0 = solve_field(rho0, rho_bar, mesh)
    _, kin_p = default_params(cfg, mesh, E0)
    row = np.empty((cfg.ng + 1, mesh.nx))
    row[0] = rho0
    for n in range(1, cfg.ng + 1):
        row[n], _ = _fine_window(n, row[n - 1], g0, cfg, kin_p, mesh, rho_bar)
    return row


@dataclass(frozen=True)
class PerfModel:
    t_hmm: float
    t_fluid: float
    t_lift: float
    n_workers: int
    ng: int
    k: int

    def __post_init__(self):
        if min(self.t_hmm, self.t_fluid, self.t_lift) < 0.0:
            raise ValueError("phase times must be nonnegative")
        if self.n_workers < 1 or self.ng < 1:
            raise ValueError("n_workers and ng must be >= 1")


def predict_cost(pm: PerfModel):
    """parareal.py:438-452."""
    per_iter = (pm.t_lift + pm.t_hmm + pm.t_fluid) / pm.n_workers + pm.t_fluid
    t_parareal = pm.t_fluid + pm.ng * pm.k * per_iter
    denom = pm.ng * per_iter
    k_opt = math.ceil((pm.ng * pm.t_hmm - pm.t_fluid) / denom) if denom > 0.0 else 0
    return t_parareal, k_opt, t_parareal <= pm.ng * pm.t_hmm
