"""Fast scan mode (``pk.scan_mode(False)``): every field solve uses a parallel
prefix sum instead of np.cumsum's sequential chain (poisson.py:52-53), so
results are no longer bitwise.  The north star's bar for it: kinetic/fluid
masks and parareal iteration counts identical, rho/E/g within 1e-10 relative
L2 (fp64) of the reference -- checked here against the same fixtures the
exact mode matches bit for bit."""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

pk = pytest.importorskip("paper_2511_13386_b200")
from paper_2511_13386_b200 import configs  # noqa: E402
import paper_2511_13386_b200.parareal as ppl  # noqa: E402

TOL = 1e-10   # relative L2, BASELINE.json north star


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("nx", [16, 100, 256, 1000, 2048, 3000, 8192])
def test_fast_coarse_chain_vs_exact(nx):
    """G (fluid_propagate) over a few hundred coarse steps, fast vs exact."""
    m = pk.build_mesh(pk.MeshSpec(nx=nx, nvx=8))
    x = m.x_centers
    rho = 1.0 + 0.3 * np.cos(x) + 0.05 * np.sin(3.0 * x)
    rb = float(rho.sum() * m.dx / m.x_star)
    p = pk.FluidStepParams.default(m)
    E0 = pk.solve_field(rho, rb, m)
    st = pk.MacroState(rho, E0, 0.0)
    t_end = min(0.2, 300.5 * p.dt)   # (long enough at small nx and rho is uniform: E == 0)
    ex = pk.fluid_propagate(st, t_end, p, m, rb)
    with pk.scan_mode(False):
        fa = pk.fluid_propagate(st, t_end, p, m, rb)
        Ef = pk.solve_field(rho, rb, m)
    assert rel(fa.rho, ex.rho) < TOL and rel(fa.E, ex.E) < TOL
    assert rel(Ef, E0) < TOL
    # fluid_step (E given on entry) through the same kernel
    with pk.scan_mode(False):
        s1 = pk.fluid_step(st, p, m, rb)
    s0 = pk.fluid_step(st, p, m, rb)
    assert rel(s1.rho, s0.rho) < TOL


def test_fast_guard_still_trips(gold):
    d = gold("field")
    m = pk.build_mesh(pk.MeshSpec(nx=64, nvx=8))
    with pk.scan_mode(False), pytest.raises(pk.SolvabilityViolation):
        pk.solve_field(d["guard_rho"], 2.0, m)


def test_fast_cfg2_parareal(gold):
    """BASELINE cfg2: same iteration count and status as the reference, every
    ledger row within 1e-10 relative L2."""
    d = gold("parareal")
    c = configs.cfg2()
    cfg = pk.PararealConfig(eps=1e-2, t_final=0.5, ng=16, k_max=5, tol=1e-10,
                            options=pk.HybridOptions(adaptation=False))
    with pk.scan_mode(False):
        res = pk.run(cfg, c.rho, c.g, c.mesh, c.rho_bar)
    assert res.iterations == int(d["c2_meta"][0]) and res.status == "converged"
    rows = np.stack(res.ledger.rho)
    assert rows.shape == d["c2_rows"].shape
    for k in range(rows.shape[0]):
        assert rel(rows[k], d["c2_rows"][k]) < TOL, k


@pytest.mark.parametrize("overlap", [True, False])
def test_fast_cfg3_iteration1(gold, monkeypatch, overlap):
    """BASELINE cfg3 iteration 1 (relaxed guard): every window's kinetic
    fraction identical, F and the jumps within 1e-10; the reference guard
    still trips in window 2 and the relaxed correction in the oracle's window."""
    d = gold("cfg3_iter1")
    monkeypatch.setattr(ppl, "OVERLAP", overlap)
    c = configs.cfg3()
    cfg = pk.PararealConfig(eps=c.eps, t_final=1.0, ng=32, k_max=50, tol=1e-8,
                            thresholds=pk.Thresholds(1e-3, 1e-3),
                            options=pk.HybridOptions(adaptation=True))
    trips = d["ref_trip"]
    first = min(n + 1 for n in range(32) if trips[n, 0] >= 0)
    with pk.scan_mode(False):
        with pytest.raises(pk.SolvabilityViolation, match=f"window {first}, step"):
            pk.run(cfg, c.rho, c.g, c.mesh, c.rho_bar)
        monkeypatch.setattr(ppl, "ADAPTIVE_FIELD_RTOL", float(d["relaxed"]))
        m = c.mesh
        E0 = pk.solve_field(c.rho, c.rho_bar, m)
        fluid_p, kin_p = ppl.default_params(cfg, m, E0)
        eng = ppl._Engine(cfg, m, c.rho, c.g, c.rho_bar, fluid_p, kin_p)
        eng.coarse_sweep()
        F, kc = eng.be.fine(eng.row[0:32], list(range(1, 33)))
        delta = eng.be.jump(F, eng.G[1:])
        assert rel(eng.row.cpu().numpy(), d["row0"]) < TOL
        assert np.array_equal(kc.cpu().numpy() / m.nx, d["frac"])
        Fh, Dh = F.cpu().numpy(), delta.cpu().numpy()
        for n in range(32):
            assert rel(Fh[n], d["F"][n]) < TOL, n
        assert rel(Dh, d["delta"]) < 1e-6   # jumps are differences of near-equal rows
        with pytest.raises(pk.SolvabilityViolation,
                           match=f"correction, window {int(d['corr_trip'])}"):
            pk.run(cfg, c.rho, c.g, m, c.rho_bar)


def test_fast_cfg4_hybrid_window_vs_oracle():
    """BASELINE cfg4's grid (8192 x 256, eps(x)), lifted restart, 12 hybrid
    steps: masks identical to the (bitwise-pinned) oracle, rho/E/g within 1e-10."""
    c = configs.cfg4()
    m = c.mesh
    grid = O.make_grid(m.nx, m.nv, v_star=10.0)
    prof = O.EpsProfile.from_function(configs.eps_bump, grid)
    rho, rb = c.rho, c.rho_bar
    E = O.field(rho, rb, grid, 1e-5)
    g = O.lift(rho, E, prof, grid, order=2, time_elim="leading", rho_bar=rb)
    dt = O.stable_dt(grid, prof, e_max=float(np.abs(E).max()))
    st = O.HState.start(rho, E, g, 0.0)
    ref = O.hpropagate(st, 12 * dt, dt, prof, 1e-3, 1e-3, O.HOpts(), grid, rb, 1e-5)
    with pk.scan_mode(False):
        E_d = pk.solve_field(rho, rb, m, rtol=1e-5)
        g_d = pk.lift(rho, E_d, c.eps, m, order=2, time_elim="leading", rho_bar=rb)
        s0 = pk.HybridState.initial(pk.MacroState(rho, E_d, 0.0), g_d, m)
        out = pk.hybrid_propagate(s0, 12 * dt, pk.KineticStepParams(eps=c.eps, dt=dt),
                                  pk.Thresholds(1e-3, 1e-3), pk.HybridOptions(), m, rb,
                                  field_rtol=1e-5)
    assert np.array_equal(out.labels.kinetic_cells, ref.kc)
    assert np.array_equal(out.labels.kinetic_ifaces, ref.ki)
    assert rel(out.macro.rho, ref.rho) < TOL and rel(out.macro.E, ref.E) < TOL
    assert rel(out.micro.g.reshape(m.nx, m.nv), ref.g) < TOL


def test_fast_kinetic_cfg1(gold):
    d = gold("kinetic")
    c = configs.cfg1()
    m = c.mesh
    st = (pk.MacroState(c.rho, np.zeros(m.nx), 0.0), pk.MicroState(c.g))
    with pk.scan_mode(False):
        mac, mic = pk.kinetic_propagate(st, 0.2, pk.KineticStepParams(eps=1.0, dt=1e-3), m,
                                        c.rho_bar)
    assert rel(mac.rho, d["c1_rho"]) < TOL and rel(mac.E, d["c1_E"]) < TOL
    assert rel(mic.g.reshape(128, 64), d["c1_g"]) < TOL
