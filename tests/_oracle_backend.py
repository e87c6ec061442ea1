"""CPU backend for the parareal engine built on the oracle (TEST ONLY).

Implements the five engine primitives of
paper_2511_13386_b200.parareal.DeviceBackend with the numpy restatement, on
CPU torch tensors, so the engine's coordination logic (window dealing across
ranks, the all-gather, the cached-G correction) can run under a gloo process
group without a GPU."""

import time

import numpy as np
import torch

import oracle as O
from paper_2511_13386_b200.errors import NonFiniteState, raise_for


class OracleBackend:
    def __init__(self, eng):
        self.eng = eng
        m = eng.mesh
        self.grid = O.make_grid(m.nx, eng.nv, x_star=m.x_star, v_star=m.v_star)
        cfg = eng.cfg
        self.pcfg = O.PConfig(eps=cfg.eps, t_final=cfg.t_final, ng=cfg.ng, k_max=cfg.k_max,
                              tol=cfg.tol, delta0=cfg.thresholds.delta0,
                              eta0=cfg.thresholds.eta0,
                              opts=O.HOpts(**cfg.options.__dict__))
        self.g0 = np.asarray(eng.g0, float).reshape(m.nx, eng.nv)

    def tensor(self, a):
        return torch.from_numpy(np.array(a, dtype=float))

    def _G(self, x, n, rtol):
        b = self.eng.cfg.boundaries
        out, _ = O.fluid_advance(x, float(b[n - 1]), float(b[n]), self.eng.fluid_p.dt, self.grid,
                                 self.eng.rho_bar, rtol)
        return out

    def chain(self, x, n0, n1, delta, rtol):
        x = x.numpy().copy()
        out, gout = [], []
        for j, n in enumerate(range(n0, n1 + 1)):
            gx = self._G(x, n, rtol)
            gout.append(gx)
            x = gx + delta[j].numpy() if delta is not None else gx
            out.append(x)
        return torch.from_numpy(np.stack(out)), torch.from_numpy(np.stack(gout))

    def many(self, X, windows, rtol):
        return torch.from_numpy(np.stack([self._G(X[j].numpy(), n, rtol)
                                          for j, n in enumerate(windows)]))

    def fine(self, X, windows):
        rows, counts = [], []
        for j, n in enumerate(windows):
            try:
                r, frac = O.fine_window(n, X[j].numpy(), self.g0, self.pcfg, self.eng.kin_p.dt,
                                        self.grid, self.eng.rho_bar)
            except O.OracleSolvability as ex:   # as the device reports it: lowest slice
                raise_for(1, str(ex), j, None)
            except O.OracleNonFinite as ex:
                raise_for(2, str(ex), j, None)
            rows.append(r)
            counts.append(int(round(frac * self.eng.nx)))
        return torch.from_numpy(np.stack(rows)), torch.tensor(counts, dtype=torch.int64)

    def jump(self, F, G):
        d = F - G
        if not torch.isfinite(d).all():
            raise NonFiniteState("non-finite fine/coarse jump (blow-up)")
        return d

    def maxdiff(self, a, b):
        if not torch.isfinite(a).all():
            raise NonFiniteState("non-finite density after parareal iteration")
        return float((a - b).abs().max())

    def clock(self):
        return time.perf_counter()

    @staticmethod
    def seconds(a, b):
        return b - a


def oracle_solve_field(grid_of):
    """A drop-in solve_field replacement backed by the oracle."""
    def solve(rho, rho_bar, mesh, rtol=None):
        return O.field(np.asarray(rho, float), rho_bar, grid_of(mesh), rtol)
    return solve
