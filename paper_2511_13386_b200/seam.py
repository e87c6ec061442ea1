"""Reference-side seam binding: the B200 fine propagator under the
reference's OWN parareal engine.

The reference's plugin seam for F is the module attribute
``parakin.parareal._fine_window(n, rho_in, g0, cfg, kin_p, mesh, rho_bar,
ws=None) -> (rho_out, {"lift_s", "fine_s", "kinetic_fraction"})``
(parareal.py:153-190), which its own tests replace with monkeypatch
(tests/test_parareal.py:54-61,124-128).  :func:`install` replaces it with
:func:`fine_window_for` bound to the reference module; every call maps the
REFERENCE's argument objects (its ``PhaseMesh``, ``PararealConfig``,
``KineticStepParams``; duck-typed, nothing is imported from the reference)
onto the drop-in's and runs the window on the device:

* mesh: ``mesh.spec`` (nx, nvx, nvy, nvz, x*, v*; mesh.py:47-65) ->
  the drop-in's ``build_mesh`` -- the reference's grids are 1D-x/3D-v with
  nvy, nvz >= 4; the resulting M, xi, dv3, m0, m2 are checked bit for bit
  against the reference mesh once per mesh object (ValueError otherwise);
* g0: the reference's (nx, nvx, nvy, nvz) array, any layout-compatible shape;
* cfg: eps (scalar or an eps(x) profile), boundaries, thresholds, options;
* the field guard: the REFERENCE module's ``field_guard(cfg)`` (so relaxing
  ``parakin.parareal.ADAPTIVE_FIELD_RTOL`` relaxes the device run too).

    import parakin.parareal as ppl
    from paper_2511_13386_b200 import seam
    seam.install(ppl)          # ppl._fine_window now runs on the B200
    ...
    seam.uninstall(ppl)
"""

from __future__ import annotations

import time

import numpy as np

from .adaptation import Thresholds
from .hybrid import HybridOptions, HybridState, hybrid_propagate
from .kinetic import KineticStepParams
from .lifting import lift
from .mesh import MacroState, MeshSpec, MicroState, build_mesh
from .poisson import solve_field

_MESHES: dict = {}   # id(reference mesh) -> (reference mesh, drop-in mesh)


def mesh_from_reference(ref_mesh):
    """The drop-in mesh of a reference ``PhaseMesh`` (cached per object),
    verified bit for bit against the reference's velocity grid."""
    hit = _MESHES.get(id(ref_mesh))
    if hit is not None and hit[0] is ref_mesh:
        return hit[1]
    sp = ref_mesh.spec
    m = build_mesh(MeshSpec(nx=int(sp.nx), nvx=int(sp.nvx), nvy=int(sp.nvy), nvz=int(sp.nvz),
                            x_star=float(sp.x_star), v_star=float(sp.v_star)))
    rg, g = ref_mesh.vgrid, m.vgrid
    same = (np.array_equal(np.asarray(rg.M).reshape(-1), np.asarray(g.M).reshape(-1))
            and np.array_equal(np.asarray(rg.vx), np.asarray(g.vx))
            and float(rg.dv3) == float(g.dv3) and float(rg.m0) == float(g.m0)
            and float(rg.m2) == float(g.m2) and float(ref_mesh.dx) == float(m.dx)
            and tuple(np.shape(rg.M)) == tuple(g.shape))
    if not same:
        raise ValueError("reference mesh does not match the drop-in's build_mesh for its spec")
    _MESHES[id(ref_mesh)] = (ref_mesh, m)
    return m


def _options(opts):
    if isinstance(opts, HybridOptions):
        return opts
    return HybridOptions(adaptation=bool(opts.adaptation), combine=opts.combine,
                         scale_remainder=bool(opts.scale_remainder), reinit=opts.reinit,
                         lift_order=opts.lift_order, time_elim=opts.time_elim)


def fine_window_for(ref_parareal):
    """F with the reference seam's signature, for the reference module
    ``ref_parareal`` (parakin.parareal)."""

    def _fine_window(n, rho_in, g0, cfg, kin_p, mesh, rho_bar, ws=None):
        m = mesh_from_reference(mesh)
        bounds = cfg.boundaries
        t0, t1 = float(bounds[n - 1]), float(bounds[n])
        rtol = ref_parareal.field_guard(cfg)
        opts = _options(cfg.options)
        th = Thresholds(float(cfg.thresholds.delta0), float(cfg.thresholds.eta0))
        rho_in = np.asarray(rho_in, dtype=float)
        E = solve_field(rho_in, rho_bar, m, rtol=rtol)
        tic = time.perf_counter()
        if n == 1:
            micro = MicroState(g=np.asarray(g0, dtype=float).reshape((m.nx,) + m.vgrid.shape))
        else:
            micro = lift(rho_in, E, cfg.eps, m, order=opts.lift_order,
                         time_elim=opts.time_elim, rho_bar=rho_bar)
        t_lift = time.perf_counter() - tic
        state = HybridState.initial(MacroState(rho=rho_in, E=E, t=t0), micro, m)
        p = KineticStepParams(eps=kin_p.eps, dt=float(kin_p.dt))
        tic = time.perf_counter()
        out = hybrid_propagate(state, t1, p, th, opts, m, rho_bar, field_rtol=rtol)
        return out.macro.rho, {"lift_s": t_lift, "fine_s": time.perf_counter() - tic,
                               "kinetic_fraction": out.labels.kinetic_fraction}

    _fine_window.__doc__ = "B200 fine window (paper_2511_13386_b200.seam) for parakin's seam"
    return _fine_window


def install(ref_parareal):
    """Replace ``ref_parareal._fine_window`` (what the reference's tests do
    with monkeypatch); the original is kept for :func:`uninstall`."""
    if not hasattr(ref_parareal, "_b200_original_fine_window"):
        ref_parareal._b200_original_fine_window = ref_parareal._fine_window
    ref_parareal._fine_window = fine_window_for(ref_parareal)
    return ref_parareal._fine_window


def uninstall(ref_parareal):
    if hasattr(ref_parareal, "_b200_original_fine_window"):
        ref_parareal._fine_window = ref_parareal._b200_original_fine_window
        del ref_parareal._b200_original_fine_window
