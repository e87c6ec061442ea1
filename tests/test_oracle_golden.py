"""Pin the CPU oracle to the real reference: every golden vector produced by
tests/golden/make_golden.py (which runs /root/reference's parakin) must be
reproduced bit for bit by the numpy restatement in oracle/."""

import numpy as np
import pytest

import oracle as O
from _cases import HYB_CASES, PAR_CASES, digest, f_cfg1, f_paper


def eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("nx,nv,vs", [(16, 8, 8.0), (32, 32, 8.0), (128, 64, 8.0), (256, 64, 8.0),
                                      (512, 128, 8.0), (1024, 128, 8.0), (8192, 256, 10.0),
                                      (16, 9, 8.0), (20, 12, 5.0), (64, 512, 8.0)])
def test_mesh(gold, nx, nv, vs):
    d = gold("mesh")
    k = f"{nx}_{nv}_{vs:g}"
    g = O.make_grid(nx, nv, v_star=vs)
    assert eq(g.vx, d["vx_" + k])
    assert eq(g.M, d["M_" + k])
    assert eq([g.dx, g.dvx, g.dv3, g.m0, g.m2], d["s_" + k])


@pytest.mark.parametrize("nx", [16, 128, 256, 1000, 8192])
def test_field(gold, nx):
    d = gold("field")
    assert eq(O.field(d[f"rho_{nx}"], 2.0, O.make_grid(nx, 8)), d[f"E_{nx}"])


def test_field_guard(gold):
    d = gold("field")
    assert bool(d["guard_raised"])
    with pytest.raises(O.OracleSolvability):
        O.field(d["guard_rho"], 2.0, O.make_grid(64, 8))


def test_kinetic_cfg1(gold):
    d = gold("kinetic")
    g = O.make_grid(128, 64)
    rho, g0, rb = O.decompose(f_cfg1(g.M), g)
    assert eq(rho, d["c1_rho0"]) and eq(g0, d["c1_g0"]) and rb == float(d["c1_rb"])
    r, E, gg = O.kinetic_advance(rho, g0, 0.0, 0.2, 1e-3, 1.0, g, rb)
    assert eq(r, d["c1_rho"]) and eq(E, d["c1_E"]) and eq(gg, d["c1_g"])


@pytest.mark.parametrize("eps", [0.5, 1e-4])
def test_kinetic_paper_with_remainder(gold, eps):
    d = gold("kinetic")
    g = O.make_grid(32, 32)
    rho, g0, rb = O.decompose(f_paper(g.vx, g.M, g.x_star), g)
    assert eq(rho, d["p_rho0"]) and eq(g0, d["p_g0"])
    E0 = O.field(rho, rb, g)
    dt = O.stable_dt(g, eps, e_max=float(np.abs(E0).max()))
    k = f"p_{eps:g}"
    assert eq([dt, 37.5 * dt], d[k + "_dt"])
    r, E, gg = O.kinetic_advance(rho, g0, 0.0, 37.5 * dt, dt, eps, g, rb)
    assert eq(r, d[k + "_rho"]) and eq(E, d[k + "_E"]) and eq(gg, d[k + "_g"])


@pytest.mark.parametrize("s", [0, 1])
def test_kinetic_cfg5_instance(gold, s):
    from paper_2511_13386_b200 import configs

    d = gold("kinetic")
    g = O.make_grid(1024, 128)
    case = configs.cfg5([s])[0]
    assert digest(case.rho) == str(d[f"c5_{s}_init"][0])
    assert digest(case.g.reshape(1024, 128)) == str(d[f"c5_{s}_init"][1])
    rb, eps, dt = d[f"c5_{s}_par"]
    assert case.rho_bar == rb and case.eps == eps
    E0 = O.field(case.rho, rb, g)
    assert O.stable_dt(g, eps, e_max=float(np.abs(E0).max())) == dt
    r, E, gg = O.kinetic_steps(case.rho, case.g.reshape(1024, 128), 5, dt, eps, g, rb)
    assert eq(r, d[f"c5_{s}_rho"]) and eq(E, d[f"c5_{s}_E"])
    assert digest(gg) == str(d[f"c5_{s}_g"])


def hyb_inputs(d, name, nx, nv):
    v = d["h_" + name + "_in"]
    n = nx * nv
    return v[:nx], v[nx:nx + n].reshape(nx, nv), v[nx + n], v[nx + n + 1], v[nx + n + 2]


@pytest.mark.parametrize("case", HYB_CASES, ids=[c[0] for c in HYB_CASES])
def test_hybrid(gold, case):
    name, data, nx, nv, eps, d0, e0, kw, nsteps, rtol = case
    d = gold("hybrid")
    rho, g0, rb, dt, t_end = hyb_inputs(d, name, nx, nv)
    grid = O.make_grid(nx, nv)
    E0 = O.field(rho, rb, grid)
    assert O.stable_dt(grid, eps, e_max=float(np.abs(E0).max())) == dt
    opts = O.HOpts(**kw)
    trace = []
    st = O.HState.start(rho, E0, g0)
    k = "h_" + name
    if k + "_raised" in d.files:
        with pytest.raises(O.OracleSolvability):
            O.hpropagate(st, t_end, dt, eps, d0, e0, opts, grid, rb, rtol,
                         trace=lambda s: trace.append(s.kc.copy()))
        assert len(trace) == int(d[k + "_raised"])
        return
    out = O.hpropagate(st, t_end, dt, eps, d0, e0, opts, grid, rb, rtol,
                       trace=lambda s: trace.append(s.kc.copy()))
    assert eq(np.array(trace), d[k + "_trace"])
    assert eq(out.rho, d[k + "_rho"]) and eq(out.E, d[k + "_E"]) and eq(out.g, d[k + "_g"])
    assert eq(out.kc, d[k + "_kc"]) and eq(out.ki, d[k + "_ki"])
    assert eq(out.E_prev, d[k + "_Eprev"])


def test_lift(gold):
    d = gold("lift")
    grid = O.make_grid(64, 32)
    rho, E, E_prev, rb = d["rho"], d["E"], d["E_prev"], float(d["rb"])
    for eps in (0.5, 1e-3):
        for order in (1, 2):
            for te in ("leading", "higher_order"):
                for proj in (True, False):
                    g = O.lift(rho, E, eps, grid, order=order, time_elim=te, rho_bar=rb,
                               dE_dt=(E - E_prev) / 1e-4, project=proj)
                    assert eq(g, d[f"l_{eps:g}_{order}_{te}_{int(proj)}"]), (eps, order, te, proj)


def test_fluid(gold):
    d = gold("fluid")
    grid = O.make_grid(256, 64)
    assert O.fluid_dt(grid) == float(d["dt"])
    r, E = O.fluid_advance(d["rho0"], 0.0, 0.5 / 16, float(d["dt"]), grid, float(d["rb"]))
    assert eq(r, d["rho"]) and eq(E, d["E"])


@pytest.mark.parametrize("case", PAR_CASES, ids=[c[0] for c in PAR_CASES])
def test_parareal_small(gold, case):
    name, nx, nv, eps, adapt, ng, T, kmax, tol, d0, e0 = case
    d = gold("parareal")
    grid = O.make_grid(nx, nv)
    rho, g0, rb = O.decompose(f_paper(grid.vx, grid.M, grid.x_star), grid)
    cfg = O.PConfig(eps=eps, t_final=T, ng=ng, k_max=kmax, tol=tol, delta0=d0, eta0=e0,
                    opts=O.HOpts(adaptation=adapt))
    k = f"p_{name}"
    if k + "_raised" in d.files:
        with pytest.raises(O.OracleSolvability):
            O.parareal(cfg, rho, g0, grid, rb)
        return
    res = O.parareal(cfg, rho, g0, grid, rb)
    assert eq(np.stack(res.rows), d[k + "_rows"])
    assert eq(res.err, d[k + "_err"])
    assert eq(res.kinetic_fraction, d[k + "_frac"])
    assert [res.iterations, res.status == "converged"] == list(d[k + "_meta"])
    if not adapt:
        assert eq(O.lift_restart_chain(cfg, rho, g0, grid, rb), d[k + "_chain"])


def test_parareal_cfg2_full(gold):
    """BASELINE cfg2 through the oracle: 4 iterations, every ledger row bitwise."""
    from paper_2511_13386_b200 import configs

    d = gold("parareal")
    case = configs.cfg2()
    grid = O.make_grid(256, 64)
    g0 = case.g.reshape(256, 64)
    assert eq(case.rho, d["c2_rho0"]) and digest(g0) == str(d["c2_g0"])
    cfg = O.PConfig(eps=1e-2, t_final=0.5, ng=16, k_max=5, tol=1e-10,
                    opts=O.HOpts(adaptation=False))
    res = O.parareal(cfg, case.rho, g0, grid, case.rho_bar)
    assert res.iterations == int(d["c2_meta"][0]) == 4
    assert eq(np.stack(res.rows), d["c2_rows"])
    assert eq(res.err, d["c2_err"])


def test_eps_profile_constant_reduces_to_scalar():
    """The eps(x) extension with a constant profile is the reference, bitwise."""
    grid = O.make_grid(48, 16)
    rho, g0, rb = O.decompose(f_paper(grid.vx, grid.M, grid.x_star), grid)
    E0 = O.field(rho, rb, grid)
    prof = O.EpsProfile.constant(1e-3, 48)
    g_l = O.lift(rho, E0, 1e-3, grid, rho_bar=rb)
    assert eq(O.lift(rho, E0, prof, grid, rho_bar=rb), g_l)
    dt = O.stable_dt(grid, 1e-3, e_max=float(np.abs(E0).max()))
    st = O.HState.start(rho, E0, g_l)
    a = O.hpropagate(st, 40.5 * dt, dt, 1e-3, 1e-2, 1e-2, O.HOpts(combine="and"), grid, rb, 1e-2)
    b = O.hpropagate(st, 40.5 * dt, dt, prof, 1e-2, 1e-2, O.HOpts(combine="and"), grid, rb, 1e-2)
    assert eq(a.rho, b.rho) and eq(a.g, b.g) and eq(a.kc, b.kc)


def test_eps_hybrid_cfg3_window2(gold):
    """eps(x) fixture (made by the oracle, tests/golden/make_eps_golden.py) is
    reproducible: the rtol-1e-5 guard trips at the recorded step of cfg3's
    window 2, and the relaxed-guard state after 600 steps matches."""
    import sys

    sys.path.insert(0, __import__("os").path.join(__import__("os").path.dirname(__file__), "golden"))
    import make_eps_golden as M

    d = gold("eps_hybrid")
    g, eps, cfg, rb, dt_c, dt_f, rho1, E1, g1 = M.window2_start()
    assert dt_f == d["dt_f"] and dt_c == d["dt_c"] and np.array_equal(rho1, d["rho1"])
    st = O.restate.HState.start(rho1, E1, g1, 0.0)
    for s in range(int(d["guard_step"])):
        st = O.restate.hstep(st, dt_f, eps, cfg.delta0, cfg.eta0, cfg.opts, g, rb, cfg.rtol)
    with pytest.raises(O.restate.OracleSolvability):
        O.restate.hstep(st, dt_f, eps, cfg.delta0, cfg.eta0, cfg.opts, g, rb, cfg.rtol)


@pytest.mark.parametrize("s", [0, 25])
def test_cfg5_500_steps_vs_reference(gold, s):
    """BASELINE cfg5 at the bench's length (500 steps): instance 0 and instance
    25, which the reference's own stable dt lets blow up (step 406)."""
    from _cases import cdigest
    from paper_2511_13386_b200 import configs

    d = gold("cfg5_500")
    c = configs.cfg5([s])[0]
    grid = O.make_grid(1024, 128)
    E0 = O.field(c.rho, c.rho_bar, grid)
    dt = O.stable_dt(grid, c.eps, e_max=float(np.abs(E0).max()))
    assert dt == d["dt"][s] and c.rho_bar == d["rho_bar"][s]
    with np.errstate(all="ignore"):
        r, E, gg = O.kinetic_steps(c.rho, c.g.reshape(1024, 128), 500, dt, c.eps, grid, c.rho_bar)
    assert cdigest(r) == d["rho_digest"][s]
    assert cdigest(E) == d["E_digest"][s]
    assert cdigest(gg) == d["g_digest"][s]
    assert np.isfinite(r).all() == (d["blowup_step"][s] < 0)
