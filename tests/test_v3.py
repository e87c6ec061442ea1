"""1D-3V grids (the reference's own mesh family, nvy, nvz >= 4) against golden
vectors from the real reference (tests/golden/make_3v_golden.py): host mesh
and brackets on CPU; kinetic steps, lift, hybrid steps with adaptation and a
parareal run on the B200, bitwise."""

import os

import numpy as np
import pytest

from _cases import digest

import paper_2511_13386_b200 as pk

MESHES = [(16, 8, 4, 4), (12, 7, 4, 4), (10, 6, 5, 4), (16, 16, 4, 4),
          (32, 32, 16, 16), (16, 17, 8, 8), (12, 30, 8, 4)]


def key(spec):
    return "_".join(str(v) for v in spec)


def mesh(spec):
    nx, nvx, nvy, nvz = spec
    return pk.build_mesh(pk.MeshSpec(nx=nx, nvx=nvx, nvy=nvy, nvz=nvz))


def initial(m):
    """experiment.py:64-85 for f0 = M xi^4 (1 + 0.9 cos(2 pi x / x*))."""
    grid = m.vgrid
    w = grid.xi**4 * grid.M

    def f(x):
        return w[None] * (1.0 + 0.9 * np.cos(2.0 * np.pi * x / m.x_star))[:, None, None, None]

    rho = m.bracket_x(f(m.x_centers))
    f_if = f(m.x_interfaces)
    g0 = f_if - m.bracket_x(f_if)[:, None, None, None] * grid.M[None]
    return rho, g0, float(rho.sum() * m.dx / m.x_star)


@pytest.mark.parametrize("spec", MESHES)
def test_mesh_and_brackets_match_reference(gold, spec):
    d = gold("v3")
    k = key(spec)
    m = mesh(spec)
    g = m.vgrid
    assert np.array_equal(g.M.reshape(-1), d["M_" + k])
    assert [m.dx, g.dvx, g.dv3, g.m0, g.m2] == list(d["s_" + k])
    rho, g0, rb = initial(m)   # host brackets over the 3V fold
    assert np.array_equal(np.concatenate([rho, [rb]]), d["in_" + k])
    assert digest(g0) == str(d["g0_" + k])


@pytest.mark.gpu
@pytest.mark.parametrize("spec", MESHES)
def test_v3_kinetic_lift_hybrid_golden(gold, spec):
    d = gold("v3")
    k = key(spec)
    m = mesh(spec)
    rho, g0, rb = initial(m)
    E0 = pk.solve_field(rho, rb, m)
    for eps in (0.5, 1e-4):
        kk = f"k_{k}_{eps:g}"
        p = pk.KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
        assert p.dt == d[kk + "_dt"]
        mac, mic = pk.kinetic_propagate((pk.MacroState(rho, E0, 0.0), pk.MicroState(g0)),
                                        12.5 * p.dt, p, m, rb)
        assert np.array_equal(mac.rho, d[kk + "_rho"]) and np.array_equal(mac.E, d[kk + "_E"])
        assert digest(mic.g) == str(d[kk + "_g"])
    for te in ("leading", "higher_order"):
        dE = (E0 - 0.5 * E0) / 1e-3
        gl = pk.lift(rho, E0, 1e-2, m, order=2, dE_dt=dE, time_elim=te, rho_bar=rb)
        assert digest(gl.g) == str(d[f"l_{k}_{te}"])
    for name, eps, start_lift, th, opts in (
            ("and", 1e-3, True, pk.Thresholds(1e-2, 1e-2), pk.HybridOptions(combine="and")),
            ("or", 0.5, False, pk.Thresholds(1e-2, 1e-2), pk.HybridOptions())):
        hk = f"h_{k}_{name}"
        p = pk.KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
        assert p.dt == d[hk + "_dt"]
        gs = pk.lift(rho, E0, eps, m, order=2, rho_bar=rb).g if start_lift else g0
        st = pk.HybridState.initial(pk.MacroState(rho, E0, 0.0), pk.MicroState(gs), m)
        res = pk.hybrid_propagate(st, 40.5 * p.dt, p, th, opts, m, rb, field_rtol=1.0)
        assert np.array_equal(res.labels.kinetic_cells, d[hk + "_kc"])
        assert np.array_equal(res.labels.kinetic_ifaces, d[hk + "_ki"])
        assert np.array_equal(res.macro.rho, d[hk + "_rho"]) and np.array_equal(res.macro.E, d[hk + "_E"])
        assert np.array_equal(res.E_prev, d[hk + "_Ep"])
        assert digest(res.micro.g) == str(d[hk + "_g"])


@pytest.mark.gpu
def test_v3_parareal_golden(gold):
    d = gold("v3")
    m = mesh((16, 8, 4, 4))
    rho, g0, rb = initial(m)
    cfg = pk.PararealConfig(eps=0.5, t_final=0.2, ng=4, k_max=6, tol=1e-10,
                            options=pk.HybridOptions(adaptation=False))
    res = pk.run(cfg, rho, g0, m, rb)
    assert np.array_equal(np.stack(res.ledger.rho), d["p_rows"])
    assert np.array_equal(res.ledger.err, d["p_err"])
    assert [res.iterations, res.status == "converged"] == list(d["p_meta"])


@pytest.mark.gpu
@pytest.mark.parametrize("eps,thr", [(1e-2, 1e-2), (1e-2, 1e-3), (1e-3, 1e-3)])
def test_v3_default_grid_mixed_labels_golden(gold, eps, thr):
    """The reference's default velocity grid (32 x 16 x 16) on partly kinetic
    slices (tests/golden/make_3v_mixed_golden.py): labels mixed at 38 % / 94 %
    or shrinking to all-fluid, so the one-CTA-per-row layout runs its sparse
    (listed-row) phases and the kinetic -> fluid zeroing; bitwise."""
    from paper_2511_13386_b200.engine import Device

    d = gold("v3_mixed")
    k = f"{eps:g}_{thr:g}"
    m = mesh((32, 32, 16, 16))
    rho, _, rb = initial(m)
    E0 = pk.solve_field(rho, rb, m)
    p = pk.KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
    assert p.dt == d[k + "_dt"]
    gs = pk.lift(rho, E0, eps, m, order=2, rho_bar=rb).g
    st = pk.HybridState.initial(pk.MacroState(rho, E0, 0.0), pk.MicroState(gs), m)
    res = pk.hybrid_propagate(st, 12.5 * p.dt, p, pk.Thresholds(thr, thr), pk.HybridOptions(), m,
                              rb, field_rtol=1.0)
    if "PK_NO_BIGC" not in os.environ:  # (the A/B switch selects the warp layout)
        assert Device.for_mesh(m).last_launch()[3] in (2, 3)  # one CTA per row
    assert np.array_equal(res.labels.kinetic_cells, d[k + "_kc"])
    assert np.array_equal(res.labels.kinetic_ifaces, d[k + "_ki"])
    assert np.array_equal(res.macro.rho, d[k + "_rho"]) and np.array_equal(res.macro.E, d[k + "_E"])
    assert np.array_equal(res.E_prev, d[k + "_Ep"])
    assert digest(res.micro.g) == str(d[k + "_g"])
