"""The reference-side seam binding (paper_2511_13386_b200.seam): the B200 fine
propagator under the reference's own plugin seam ``parakin.parareal.
_fine_window`` (parareal.py:153-190).

GPU tests drive it with duck-typed stand-ins of the REFERENCE's objects (its
PhaseMesh / PararealConfig / KineticStepParams attributes, built from values
tests/golden/make_seam_golden.py recorded from the real reference -- the
reference itself does not exist on the GPU box) on the reference's default
1D-3V grid (nx=32, 32 x 16 x 16), bitwise against the reference's own
_fine_window.  CPU tests check the object mapping against the real reference
where it is importable (this container)."""

import os
import sys
import types

import numpy as np
import pytest

from _cases import digest

import paper_2511_13386_b200 as pk
from paper_2511_13386_b200 import seam

REF = "/root/reference/pkg/src"


def _duck(d, case):
    """Stand-ins with exactly the reference attributes the seam reads."""
    nx, nvx, nvy, nvz, xs, vs = d["spec"]
    dx, dv3, m0, m2 = d["vgrid"]
    spec = types.SimpleNamespace(nx=int(nx), nvx=int(nvx), nvy=int(nvy), nvz=int(nvz),
                                 x_star=float(xs), v_star=float(vs))
    vgrid = types.SimpleNamespace(M=d["M"].reshape(int(nvx), int(nvy), int(nvz)), vx=d["vx"],
                                  dv3=float(dv3), m0=float(m0), m2=float(m2))
    mesh = types.SimpleNamespace(spec=spec, vgrid=vgrid, dx=float(dx), nx=int(nx))
    eps, th = (float(x) for x in d[f"{case}_par"])
    t_final = float(d[f"{case}_t_final"])
    cfg = types.SimpleNamespace(
        eps=eps, boundaries=np.linspace(0.0, t_final, 5),
        thresholds=types.SimpleNamespace(delta0=th, eta0=th),
        options=types.SimpleNamespace(adaptation=True, combine=case, scale_remainder=False,
                                      reinit="lift", lift_order=2, time_elim="leading"))
    kin_p = types.SimpleNamespace(eps=eps, dt=float(d[f"{case}_dt"]))
    # the reference module as the seam sees it (field_guard: its relaxed 1.0)
    ref = types.SimpleNamespace(field_guard=lambda c: 1.0, _fine_window=None)
    return mesh, cfg, kin_p, ref


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["or", "and"])
def test_seam_fine_window_vs_reference(gold, case):
    d = gold("seam")
    mesh, cfg, kin_p, ref = _duck(d, case)
    m = seam.mesh_from_reference(mesh)
    # the reference's initial data on the drop-in mesh (make_3v_golden.initial)
    grid = m.vgrid
    w = grid.xi**4 * grid.M
    f = lambda x: w[None] * (1.0 + 0.9 * np.cos(2.0 * np.pi * x / m.x_star))[:, None, None, None]  # noqa: E731
    rho = m.bracket_x(f(m.x_centers))
    f_if = f(m.x_interfaces)
    g0 = f_if - m.bracket_x(f_if)[:, None, None, None] * grid.M[None]
    assert np.array_equal(rho, d["rho0"]) and digest(g0) == str(d["g0_digest"])
    fw = seam.install(ref)
    try:
        assert ref._fine_window is fw
        for n in (1, 2):
            r, diag = ref._fine_window(n, d[f"{case}_w{n}_in"], g0, cfg, kin_p, mesh,
                                       float(d["rho_bar"]))
            assert np.array_equal(r, d[f"{case}_w{n}_rho"]), n
            assert diag["kinetic_fraction"] == float(d[f"{case}_w{n}_frac"])
            assert set(diag) == {"lift_s", "fine_s", "kinetic_fraction"}
    finally:
        seam.uninstall(ref)
    assert ref._fine_window is None


@pytest.mark.gpu
def test_seam_under_the_host_engine(gold):
    """The seam function also binds to the drop-in's own seam (its objects
    carry the same attributes): the reference-order host engine then runs
    the small 1D-3V parareal golden bitwise."""
    import paper_2511_13386_b200.parareal as ppl

    d = gold("v3")
    m = pk.build_mesh(pk.MeshSpec(nx=16, nvx=8, nvy=4, nvz=4))
    grid = m.vgrid
    w = grid.xi**4 * grid.M
    f = lambda x: w[None] * (1.0 + 0.9 * np.cos(2.0 * np.pi * x / m.x_star))[:, None, None, None]  # noqa: E731
    rho = m.bracket_x(f(m.x_centers))
    f_if = f(m.x_interfaces)
    g0 = f_if - m.bracket_x(f_if)[:, None, None, None] * grid.M[None]
    rb = float(rho.sum() * m.dx / m.x_star)
    cfg = pk.PararealConfig(eps=0.5, t_final=0.2, ng=4, k_max=6, tol=1e-10,
                            options=pk.HybridOptions(adaptation=False))
    seam.install(ppl)
    try:
        res = pk.run(cfg, rho, g0, m, rb)
    finally:
        seam.uninstall(ppl)
    assert ppl._fine_window is ppl._ORIG_FINE_WINDOW
    assert np.array_equal(np.stack(res.ledger.rho), d["p_rows"])
    assert np.array_equal(res.ledger.err, d["p_err"])


@pytest.mark.skipif(not os.path.isdir(REF), reason="needs the reference (build container)")
@pytest.mark.parametrize("spec", [(32, 32, 16, 16), (16, 8, 4, 4), (12, 7, 5, 4)])
def test_seam_maps_reference_meshes(spec):
    """The mapping the round-1 INTEGRATION snippet got wrong (nvy/nvz dropped):
    every reference mesh maps onto a drop-in mesh with the same grid bits."""
    sys.path.insert(0, REF)
    from parakin.mesh import MeshSpec, build_mesh

    nx, nvx, nvy, nvz = spec
    rm = build_mesh(MeshSpec(nx=nx, nvx=nvx, nvy=nvy, nvz=nvz))
    m = seam.mesh_from_reference(rm)
    assert m.vgrid.shape == rm.vgrid.M.shape == (nvx, nvy, nvz)
    assert np.array_equal(m.vgrid.M, rm.vgrid.M) and np.array_equal(m.xi_M, rm.xi_M)
    assert seam.mesh_from_reference(rm) is m          # cached per reference object
    g = np.zeros((nx, nvx, nvy, nvz))
    assert g.reshape((m.nx,) + m.vgrid.shape).shape == g.shape


@pytest.mark.skipif(not os.path.isdir(REF), reason="needs the reference (build container)")
def test_seam_install_on_reference_module():
    sys.path.insert(0, REF)
    import parakin.parareal as rppl

    orig = rppl._fine_window
    fw = seam.install(rppl)
    try:
        assert rppl._fine_window is fw and fw is not orig
    finally:
        seam.uninstall(rppl)
    assert rppl._fine_window is orig
