"""Batched fine-solver API: B independent slices (instances, or parareal
windows) advanced together in one persistent-kernel launch.

This is the throughput entry point the reference lacks as a single call (its
equivalent is B independent ``kinetic_step`` loops, kinetic.py:255-273, or a
process pool over instances).  Two forms:

* :class:`Ensemble` keeps the state resident on the device (``run`` advances
  every slice ``nsteps`` steps in place);
* :func:`kinetic_ensemble` is the host-array call: copies in, runs, copies out;
* :class:`EnsemblePipeline` streams host-array batches through two resident
  state sets so that the host<->device copies of one batch overlap the kernel
  of the next.
"""

from __future__ import annotations

import numpy as np

from .engine import Device, HybridKnobs, make_phase
from .kinetic import KineticStepParams
from .mesh import PhaseMesh
from .poisson import SOLVABILITY_RTOL


class Ensemble:
    """Device-resident batch of B slices on one mesh."""

    def __init__(self, mesh: PhaseMesh, eps, dt, rho_bar, device=None):
        import torch

        self.torch = torch
        self.mesh = mesh
        self.dev = Device.for_mesh(mesh, device)
        self.B = len(eps)
        self.eps = list(eps)
        self.dt = [float(x) for x in dt]
        for e, h in zip(self.eps, self.dt):
            KineticStepParams(eps=e, dt=h).check(h, mesh)
        nx, nv = mesh.nx, mesh.nv
        d = self.dev.device
        self.rho = torch.empty((self.B, nx), dtype=torch.float64, device=d)
        self.E = torch.zeros_like(self.rho)
        self.Ep = torch.zeros_like(self.rho)
        self.g = torch.empty((self.B, nx, nv), dtype=torch.float64, device=d)
        self.kc = torch.ones((self.B, nx), dtype=torch.uint8, device=d)
        self.ki = torch.ones_like(self.kc)
        self.rb = self.dev.t(np.asarray(rho_bar, dtype=float).reshape(self.B))
        self.flags = self.dev.t(np.zeros(self.B, dtype=np.uint8))  # plain kinetic steps
        self._prep = {}
        self.dev.reserve(self.B)
        self.dev.scratch("gb", (self.B, nx, nv))

    def load(self, rho, g, non_blocking=False):
        """Copy inputs (host or device arrays) into the resident state."""
        torch = self.torch
        for dst, src in ((self.rho, rho), (self.g, g)):
            if isinstance(src, torch.Tensor):
                dst.copy_(src.reshape(dst.shape), non_blocking=non_blocking)
            else:
                dst.copy_(torch.from_numpy(np.ascontiguousarray(src).reshape(dst.shape)),
                          non_blocking=non_blocking)

    def prepared(self, nsteps):
        from . import engine

        key = (nsteps, engine.EXACT)
        p = self._prep.get(key)
        if p is None:
            ph0 = make_phase(self.mesh, self.eps, self.dt, [nsteps] * self.B)
            ph1 = make_phase(self.mesh, self.eps, self.dt, [0] * self.B)
            p = self._prep[key] = ((ph0, ph1),
                                   self.dev.prepare_fine(self.B, [ph0, ph1], HybridKnobs(),
                                                         self.eps))
        return p

    def run(self, nsteps: int, check: bool = True):
        """Advance every slice ``nsteps`` kinetic steps (kinetic.py:255-273)."""
        phases, prep = self.prepared(nsteps)
        self.dev.fine(self.rho, self.E, self.Ep, self.kc, self.ki, self.g, self.rb,
                      self.flags, phases, HybridKnobs(), self.eps, SOLVABILITY_RTOL,
                      prepared=prep)
        if check:
            self.dev.check()


def kinetic_ensemble(mesh: PhaseMesh, rho, g, eps, dt, rho_bar, nsteps: int):
    """Host-array batched ``nsteps`` x ``kinetic_step`` over B slices.
    rho [B, nx], g [B, nx, nv(,1,1)] -> (rho, E, g) host arrays."""
    ens = Ensemble(mesh, eps, dt, rho_bar)
    ens.load(rho, g)
    ens.run(nsteps)
    return (ens.rho.cpu().numpy(), ens.E.cpu().numpy(),
            ens.g.cpu().numpy().reshape(np.shape(g)))


class EnsemblePipeline:
    """Host-array batches through the fine solver with the copies overlapped.

    Two resident state sets alternate: batch i's upload (copy stream `h2d`)
    and the previous batch's download (copy stream `d2h`) run while batch i-1
    computes; the kernels themselves run one after another on one stream (they
    share the context's workspace).  Events order every hand-over, so results
    are those of ``kinetic_ensemble`` batch by batch.  Host buffers should be
    pinned for the copies to overlap.  While batches are in flight the pipeline
    owns the device's solver context (its workspace is shared by every solver
    call on that device and mesh): call ``drain`` before any other solver work.
    """

    def __init__(self, mesh: PhaseMesh, eps, dt, rho_bar, nsteps: int, device=None):
        import torch

        self.torch = torch
        self.nsteps = int(nsteps)
        self.sets = [Ensemble(mesh, eps, dt, rho_bar, device) for _ in range(2)]
        for s in self.sets:
            s.prepared(self.nsteps)
        d = self.sets[0].dev.device
        self.h2d, self.comp, self.d2h = (torch.cuda.Stream(d) for _ in range(3))
        ev = lambda: [torch.cuda.Event() for _ in range(2)]  # noqa: E731
        self.loaded, self.computed, self.drained = ev(), ev(), ev()
        for e in self.drained:
            e.record(self.d2h)
        self.i = 0

    def submit(self, rho, g, out_rho, out_E, out_g):
        """Enqueue one batch: rho [B, nx], g [B, nx, nv] in; results copied to
        out_* (host tensors) when the batch completes (see ``drain``)."""
        torch = self.torch
        k = self.i & 1
        s = self.sets[k]
        with torch.cuda.stream(self.h2d):
            self.h2d.wait_event(self.drained[k])    # set k's previous results are out
            s.load(rho, g, non_blocking=True)
            self.loaded[k].record(self.h2d)
        with torch.cuda.stream(self.comp):
            self.comp.wait_event(self.loaded[k])
            s.run(self.nsteps, check=False)
            self.computed[k].record(self.comp)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self.computed[k])
            out_rho.copy_(s.rho, non_blocking=True)
            out_E.copy_(s.E, non_blocking=True)
            out_g.copy_(s.g.reshape(out_g.shape), non_blocking=True)
            self.drained[k].record(self.d2h)
        self.i += 1

    def drain(self):
        """Wait for every submitted batch; raise the device status, if any."""
        for st in (self.h2d, self.comp, self.d2h):
            st.synchronize()
        self.sets[0].dev.check()
