"""Device engine: one libpk context per (CUDA device, mesh), batched entry
points on torch CUDA tensors, and the host-side formation of the scalar
constants the kernels consume.

Everything numeric that the reference forms as a Python float (kappa1/2,
dt/(eps dx), m2 (dt/dx), eps**2, dx**-p, ...) is formed here the same way and
uploaded, so the device arithmetic starts from bit-identical constants
(SURVEY F10).  torch is used only for device memory and streams.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import NativeError, raise_for
from .mesh import PhaseMesh

STENCIL_COEFFS = {  # adaptation.py:29-34 (Python floats)
    1: (-1 / 60, 3 / 20, -3 / 4, 0.0, 3 / 4, -3 / 20, 1 / 60),
    2: (1 / 90, -3 / 20, 3 / 2, -49 / 18, 3 / 2, -3 / 20, 1 / 90),
    3: (1 / 8, -1.0, 13 / 8, 0.0, -13 / 8, 1.0, -1 / 8),
    4: (-1 / 6, 2.0, -13 / 2, 28 / 3, -13 / 2, 2.0, -1 / 6),
}


# Scan mode of every field solve (coarse G, the fine kernels' slice phase and
# the standalone solve_field).  True (default): np.cumsum's sequential order,
# bitwise equal to the reference.  False ("fast"): a parallel prefix sum --
# results differ from the reference by O(nx u |E|) per solve (north star:
# masks and iteration counts identical, rho/E/g within 1e-10 relative L2),
# the coarse step at nx = 8192 drops from ~48 us to a few us.
EXACT = True


@contextlib.contextmanager
def scan_mode(exact: bool):
    """Run a block of drop-in calls in exact (bitwise) or fast scan mode."""
    global EXACT
    old, EXACT = EXACT, bool(exact)
    try:
        yield
    finally:
        EXACT = old


def _torch():
    import torch
    return torch


def _ptr(t):
    """Device pointer of a tensor for libpk, which reads every array as dense
    C order: a strided view is refused loudly rather than misread."""
    if t is None:
        return C.c_void_p(0)
    if not t.is_contiguous():
        raise NativeError(f"libpk needs contiguous arrays (got strides {t.stride()})")
    return C.c_void_p(t.data_ptr())


def relaxation_coefficients(dt: float, eps: float):
    """(e^{-dt/eps^2}, eps (1 - e^{-dt/eps^2})) (kinetic.py:141-145)."""
    z = dt / eps**2
    return float(np.exp(-z)), float(eps * (-np.expm1(-z)))


@dataclass
class Phase:
    """Host description of one run of identical steps for B slices."""

    nsteps: np.ndarray   # int32 [B]
    dt: np.ndarray       # [B]
    cflu: np.ndarray     # [B]
    k1: np.ndarray       # [B, nx]
    k2: np.ndarray       # [B, nx]
    cmac: np.ndarray     # [B, nx]
    cmac_scalar: np.ndarray = None  # [B]: the common cmac when uniform in x, else NaN
    k1_scalar: np.ndarray = None    # [B]: the common kappa1 when uniform in x, else NaN
    k2_scalar: np.ndarray = None    # [B]: the common kappa2 when uniform in x, else NaN


def eps_rows(eps, nx: int) -> np.ndarray:
    """Per-interface eps values of a scalar or an EpsProfile."""
    iface = getattr(eps, "iface", None)
    if iface is not None:
        return np.asarray(iface, dtype=float)
    return np.full(nx, float(eps))


def eps_cells(eps, nx: int) -> np.ndarray:
    cell = getattr(eps, "cell", None)
    if cell is not None:
        return np.asarray(cell, dtype=float)
    return np.full(nx, float(eps))


def per_value(values: np.ndarray, fn) -> np.ndarray:
    """Apply a scalar Python-float rule once per distinct value."""
    out = np.empty(values.shape[0])
    cache = {}
    for i, e in enumerate(values.tolist()):
        r = cache.get(e)
        if r is None:
            r = cache[e] = fn(e)
        out[i] = r
    return out


_COEF_ROWS: dict = {}   # (mesh, eps, dt) -> coefficient rows (insertion-ordered LRU)
_EPS_ROWS: dict = {}    # (eps, nx, kind) -> (eps, row): -eps_i, eps_i**2, eps_c**2


def _eps_row(eps, nx: int, kind: str) -> np.ndarray:
    """-eps_i, eps_i**2 per interface or eps_c**2 per cell as Python floats per
    distinct value (per_value), memoised per eps object: a parareal run passes
    the same profile for every window."""
    key = (id(eps) if hasattr(eps, "iface") else float(eps), nx, kind)
    hit = _EPS_ROWS.get(key)
    if hit is None or (hasattr(eps, "iface") and hit[0] is not eps):
        if kind == "neg":
            row = per_value(eps_rows(eps, nx), lambda v: -v)
        elif kind == "sq":
            row = per_value(eps_rows(eps, nx), lambda v: v**2)
        else:
            row = per_value(eps_cells(eps, nx), lambda v: v**2)
        hit = _EPS_ROWS[key] = (eps, row)
        while len(_EPS_ROWS) > 64:
            _EPS_ROWS.pop(next(iter(_EPS_ROWS)))
    return hit[1]


def _coef_rows(mesh: PhaseMesh, eps, dt: float):
    """kappa1, kappa2 and dt/(eps dx) per interface for one (eps, dt): Python
    floats per distinct eps value (an eps(x) profile has nx of them, ~30 ms
    at nx = 8192), so they are cached across calls."""
    key = (id(mesh), id(eps) if hasattr(eps, "iface") else float(eps), dt)
    hit = _COEF_ROWS.pop(key, None)
    if hit is None or hit[0] is not mesh or (hasattr(eps, "iface") and hit[1] is not eps):
        e = eps_rows(eps, mesh.nx)
        dx = mesh.dx
        hit = (mesh, eps, (per_value(e, lambda v: relaxation_coefficients(dt, v)[0]),
                           per_value(e, lambda v: relaxation_coefficients(dt, v)[1]),
                           per_value(e, lambda v: dt / (v * dx))))
    _COEF_ROWS[key] = hit
    while len(_COEF_ROWS) > 64:
        _COEF_ROWS.pop(next(iter(_COEF_ROWS)))
    return hit[2]


def make_phase(mesh: PhaseMesh, eps_list, dt_list, nsteps_list) -> Phase:
    """Coefficients of a run of steps; slice b uses eps_list[b], dt_list[b]."""
    B = len(eps_list)
    nx, dx, m2 = mesh.nx, mesh.dx, mesh.vgrid.m2
    k1 = np.empty((B, nx))
    k2 = np.empty((B, nx))
    cm = np.empty((B, nx))
    cflu = np.empty(B)
    dts = np.empty(B)
    for b in range(B):
        dt = float(dt_list[b])
        dts[b] = dt
        k1[b], k2[b], cm[b] = _coef_rows(mesh, eps_list[b], dt)
        cflu[b] = m2 * (dt / dx)
    def uniform(a):  # per slice: the common value of a row, else NaN
        return np.array([row[0] if (row == row[0]).all() else np.nan for row in a])

    return Phase(np.asarray(nsteps_list, dtype=np.int32), dts, cflu, k1, k2, cm, uniform(cm),
                 uniform(k1), uniform(k2))


@dataclass
class HybridKnobs:
    adaptation: bool = False
    combine: str = "or"
    scale_remainder: bool = False
    reinit: str = "lift"
    lift_order: int = 2
    time_elim: str = "leading"
    delta0: float = 1.0
    eta0: float = 1.0


def _combine_code(c):
    if c == "or":
        return 0
    if c == "and":
        return 1
    raise ValueError(f"combine must be 'or' or 'and', got {c!r}")


class Device:
    """libpk context bound to one mesh on one CUDA device."""

    _cache: dict = {}
    _lock = threading.Lock()

    @classmethod
    def for_mesh(cls, mesh: PhaseMesh, device=None) -> "Device":
        torch = _torch()
        if not torch.cuda.is_available():
            raise NativeError("no CUDA device: the B200 engine has no CPU fallback")
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                           torch.device(device).index or 0)
        key = (dev.index, id(mesh))
        with cls._lock:
            d = cls._cache.get(key)
            if d is None or d.mesh is not mesh:
                d = cls._cache[key] = cls(mesh, dev)
            return d

    def __init__(self, mesh: PhaseMesh, device):
        torch = _torch()
        self.lib = _native.load()
        self.mesh = mesh
        self.device = torch.device(device)
        self.nx = mesh.nx
        self.nv = mesh.nv
        grid = mesh.vgrid
        # xi of every node of a row: (nvx, nvy, nvz) in C order
        vx = np.ascontiguousarray(np.repeat(np.asarray(grid.vx, dtype=float), mesh.nvyz))
        M = np.ascontiguousarray(grid.M.reshape(-1))
        xiM = np.ascontiguousarray(mesh.xi_M.reshape(-1))
        w2 = np.ascontiguousarray(((grid.xi**2 - 1.0) * grid.M).reshape(-1))
        self._keep = (vx, M, xiM, w2)
        m = _native.PkMesh()
        m.nx, m.nv = mesh.nx, self.nv
        m.dx, m.dvx, m.dv3 = mesh.dx, grid.dvx, grid.dv3
        m.m0, m.m2, m.x_star, m.v_star = grid.m0, grid.m2, mesh.x_star, mesh.v_star
        dp = lambda a: a.ctypes.data_as(_native.c_double_p)  # noqa: E731
        m.vx, m.M, m.xi_M, m.w2 = dp(vx), dp(M), dp(xiM), dp(w2)
        for p in range(4):
            for o in range(7):
                m.stencil[p][o] = STENCIL_COEFFS[p + 1][o]
            m.stencil_scale[p] = mesh.dx ** (-(p + 1))
        m.nvyz = mesh.nvyz
        with torch.cuda.device(self.device):
            torch.cuda.init()
            self.ctx = self.lib.pk_create(self.device.index or 0, C.byref(m))
        if not self.ctx:
            raise NativeError("pk_create failed (unsupported mesh or CUDA error)")
        self._scratch = {}

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx:
            try:
                self.lib.pk_destroy(ctx)
            except Exception:
                pass

    # -- helpers -------------------------------------------------------------
    @property
    def stream(self):
        torch = _torch()
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def t(self, a, dtype=None):
        """Host array -> contiguous device tensor."""
        torch = _torch()
        if isinstance(a, torch.Tensor):
            return a.to(device=self.device, dtype=dtype or a.dtype).contiguous()
        a = np.ascontiguousarray(a)
        return torch.from_numpy(a).to(self.device, non_blocking=False)

    def scratch(self, name, shape, dtype=None):
        """Named grow-only work buffer: a view of the first prod(shape)
        elements.  One buffer per (name, dtype) -- a shrinking batch (B = Ng - k
        active windows) reuses it instead of allocating per distinct shape.
        Growth synchronises the device first, so no queued kernel (on any
        stream) still uses the buffer that is dropped."""
        torch = _torch()
        dtype = dtype or torch.float64
        n = int(np.prod(shape))
        key = (name, dtype)
        buf = self._scratch.get(key)
        if buf is None or buf.numel() < n:
            if buf is not None:
                torch.cuda.synchronize(self.device)
            buf = self._scratch[key] = torch.empty(max(n, 1), dtype=dtype, device=self.device)
        return buf[:n].view(tuple(shape))

    def _rc(self, code, what):
        if code != 0:
            msg = self.lib.pk_last_error(self.ctx)
            raise_for(code, f"{what}: {msg.decode() if msg else ''}")

    def cancel(self, stream):
        """Ask the fine launch in flight on this context to stop (pk_fine_cancel);
        `stream`: a torch stream other than the launch's own."""
        self._rc(self.lib.pk_fine_cancel(self.ctx, C.c_void_p(stream.cuda_stream)), "pk_fine_cancel")

    def last_launch(self):
        """Layout of this thread's last fine launch: (CTAs per cluster or group,
        slices per cluster, slice vectors in shared memory, kind: 0 hardware
        cluster, 1 software group, 2 big rows one CTA per row in hardware clusters,
        3 the same in software groups)."""
        out = (C.c_int32 * 4)()
        self._rc(self.lib.pk_fine_last_launch(self.ctx, out), "pk_fine_last_launch")
        return out[0], out[1], bool(out[2]), int(out[3])

    def check_stream(self, stream):
        """Raise this context's latched status after the work queued on
        `stream` (a torch.cuda.Stream) -- without synchronising the device."""
        st = _native.PkStatus()
        self._rc(self.lib.pk_status_read_stream(self.ctx, C.byref(st), 1,
                                                C.c_void_p(stream.cuda_stream)), "status")
        if st.code:
            raise_for(st.code, f"slice {st.slice}, step {st.step}", st.slice, st.step)

    def check(self):
        """Synchronise and raise the latched device status, if any."""
        st = _native.PkStatus()
        self._rc(self.lib.pk_status_read(self.ctx, C.byref(st), 1), "status")
        if st.code:
            raise_for(st.code, f"slice {st.slice}, step {st.step}", st.slice, st.step)

    def count_rows(self, counts=None):
        """Measurement hook (pk_count_rows): accumulate per slice b of every
        following fine launch the rows streamed (counts[b, 0]) and zeroed
        (counts[b, 1]) into a device int64 tensor [B, 2]; None disables."""
        self._rc(self.lib.pk_count_rows(self.ctx, _ptr(counts)), "pk_count_rows")
        self._rowcnt = counts

    def reserve(self, B):
        self._rc(self.lib.pk_reserve(self.ctx, int(B)), "reserve")

    # -- entry points --------------------------------------------------------
    def phase_dev(self, ph: Phase):
        torch = _torch()
        dev = dict(
            nsteps=self.t(ph.nsteps.astype(np.int32)), dt=self.t(ph.dt), cflu=self.t(ph.cflu),
            k1=self.t(ph.k1), k2=self.t(ph.k2), cmac=self.t(ph.cmac), cs=self.t(ph.cmac_scalar),
            k1s=self.t(ph.k1_scalar), k2s=self.t(ph.k2_scalar))
        s = _native.PkPhase()
        s.nsteps, s.dt, s.cflu = _ptr(dev["nsteps"]), _ptr(dev["dt"]), _ptr(dev["cflu"])
        s.kappa1, s.kappa2, s.cmac = _ptr(dev["k1"]), _ptr(dev["k2"]), _ptr(dev["cmac"])
        s.cmac_scalar = _ptr(dev["cs"])
        s.kappa1_scalar, s.kappa2_scalar = _ptr(dev["k1s"]), _ptr(dev["k2s"])
        del torch
        return s, dev

    def fine(self, rho, E, Eprev, kc, ki, g, rho_bar, init_flags, phases, knobs: HybridKnobs,
             eps_list, rtol, exact_scan=None, cluster_hint=0, prepared=None):
        """Advance B slices in place (device tensors).  ``phases``: [full, rem]."""
        B = rho.shape[0]
        nx, nv = self.nx, self.nv
        if prepared is None:
            prepared = self.prepare_fine(B, phases, knobs, eps_list)
        ph_structs, hyb, keep = prepared
        gb = self.scratch("gb", (B, nx, nv))
        self.reserve(B)
        # a device tensor is used as is (no per-call upload: a pageable copy
        # would block the host until the stream drains)
        flags = (init_flags if isinstance(init_flags, _torch().Tensor)
                 else self.t(np.asarray(init_flags, dtype=np.uint8)))
        rc = self.lib.pk_fine_propagate(
            self.ctx, B, _ptr(rho), _ptr(E), _ptr(Eprev), _ptr(kc), _ptr(ki), _ptr(g), _ptr(gb),
            _ptr(rho_bar), _ptr(flags), ph_structs, C.byref(hyb), float(rtol),
            int(cluster_hint), self.stream)
        self._rc(rc, "pk_fine_propagate")
        self._keepalive = (keep, flags)

    def prepare_fine(self, B, phases, knobs: HybridKnobs, eps_list):
        """Upload phase coefficients and hybrid knobs (reusable across calls)."""
        nx = self.nx
        arr = (_native.PkPhase * 2)()
        keep = []
        for p in range(2):
            s, dev = self.phase_dev(phases[p])
            arr[p] = s
            keep.append(dev)
        hyb = _native.PkHybrid()
        hyb.adaptation = int(bool(knobs.adaptation))
        hyb.combine_and = _combine_code(knobs.combine) if knobs.adaptation else 0
        hyb.reinit = {"lift": 0, "zero": 1}.get(knobs.reinit, 2)
        hyb.lift_order = int(knobs.lift_order) if knobs.lift_order in (1, 2) else 0
        hyb.time_elim = {"leading": 0, "higher_order": 1}.get(knobs.time_elim, 2)
        hyb.exact_scan = int(EXACT)
        hyb.delta0, hyb.eta0 = float(knobs.delta0), float(knobs.eta0)
        neg = np.stack([_eps_row(e, nx, "neg") for e in eps_list])
        e2 = np.stack([_eps_row(e, nx, "sq") for e in eps_list])
        dneg, de2 = self.t(neg), self.t(e2)
        hyb.neg_eps, hyb.eps2 = _ptr(dneg), _ptr(de2)
        keep += [dneg, de2]
        if knobs.adaptation and knobs.scale_remainder:
            rs = self.t(np.stack([_eps_row(e, nx, "cellsq") for e in eps_list]))
            hyb.rscale = _ptr(rs)
            keep.append(rs)
        else:
            hyb.rscale = C.c_void_p(0)
        return arr, hyb, keep

    def chain(self, rho_in, out, gout, E_out, delta, nfull, rem, dt_full, rho_bar, rtol,
              exact_scan=None, E_in=None, m2=None):
        """Coarse chains: rho_in [nchain, nx], out/gout/delta [nchain, nwin, nx]."""
        nchain, nwin = out.shape[0], out.shape[1]
        nfull = np.asarray(nfull, dtype=np.int32).reshape(nchain, nwin)
        rem = np.asarray(rem, dtype=float).reshape(nchain, nwin)
        sched = self.chain_schedule(nfull, rem, dt_full, m2)
        self.chain_raw(rho_in, out, gout, E_out, delta, sched, dt_full, rho_bar, rtol, exact_scan,
                       E_in)
        self._keepalive = sched

    def chain_schedule(self, nfull, rem, dt_full, m2=None):
        """Device copies of a chain's per-window step schedule (nfull, rem and
        the cflu factors m2 dt/dx), reusable across chain_raw calls."""
        m2 = self.mesh.vgrid.m2 if m2 is None else m2
        dx = self.mesh.dx
        nfull = np.atleast_2d(np.asarray(nfull, dtype=np.int32))
        rem = np.atleast_2d(np.asarray(rem, dtype=float))
        cf = np.full(nfull.shape, m2 * (dt_full / dx))
        cr = np.vectorize(lambda r: m2 * (r / dx) if r > 0.0 else 0.0)(rem) if rem.size else rem
        return (self.t(nfull), self.t(rem), self.t(cf), self.t(np.asarray(cr, float)))

    def chain_raw(self, rho_in, out, gout, E_out, delta, sched, dt_full, rho_bar, rtol,
                  exact_scan=None, E_in=None):
        """pk_coarse_chain on the current stream with a prepared schedule (no uploads)."""
        nchain, nwin = out.shape[0], out.shape[1]
        d_nf, d_rem, d_cf, d_cr = sched
        rc = self.lib.pk_coarse_chain(
            self.ctx, nchain, nwin, _ptr(rho_in), _ptr(E_in), _ptr(out), _ptr(gout), _ptr(E_out),
            _ptr(delta),
            _ptr(d_nf), _ptr(d_rem), _ptr(d_cf), _ptr(d_cr), float(dt_full), _ptr(rho_bar),
            float(rtol), int(EXACT if exact_scan is None else bool(exact_scan)), self.stream)
        self._rc(rc, "pk_coarse_chain")

    def field(self, rho, rho_bar, E, rtol, exact_scan=None):
        self.reserve(rho.shape[0])
        rc = self.lib.pk_field(self.ctx, rho.shape[0], _ptr(rho), _ptr(rho_bar), _ptr(E),
                               float(rtol), int(EXACT if exact_scan is None else bool(exact_scan)),
                               self.stream)
        self._rc(rc, "pk_field")

    def lift(self, rho, E, dE_dt, rho_bar, eps_list, order, time_elim, project, g_out):
        B, nx = rho.shape
        self.reserve(B)
        neg = self.t(np.stack([per_value(eps_rows(e, nx), lambda v: -v) for e in eps_list]))
        e2 = self.t(np.stack([per_value(eps_rows(e, nx), lambda v: v**2) for e in eps_list]))
        te = {"leading": 0, "higher_order": 1}.get(time_elim, 2)
        rc = self.lib.pk_lift(self.ctx, B, _ptr(rho), _ptr(E), _ptr(dE_dt), _ptr(rho_bar),
                              _ptr(neg), _ptr(e2), int(order), te, int(bool(project)),
                              _ptr(g_out), self.stream)
        self._rc(rc, "pk_lift")
        self._keepalive = (neg, e2)

    def jump(self, a, b, out):
        rc = self.lib.pk_jump(self.ctx, a.numel(), _ptr(a), _ptr(b), _ptr(out), self.stream)
        self._rc(rc, "pk_jump")

    def maxdiff(self, a, b, err):
        rc = self.lib.pk_maxdiff(self.ctx, a.numel(), _ptr(a), _ptr(b), _ptr(err), self.stream)
        self._rc(rc, "pk_maxdiff")
