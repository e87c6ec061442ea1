"""Host-side logic of the drop-in (no GPU): mesh construction, BASELINE input
builders, step-size rules, schedules, error taxonomy, cost model — all against
the golden vectors of the real reference or the oracle."""

import math

import numpy as np
import pytest

import oracle as O
import paper_2511_13386_b200 as pk
from paper_2511_13386_b200 import configs, errors
from paper_2511_13386_b200.engine import make_phase, relaxation_coefficients
from paper_2511_13386_b200.fluid import substep_sizes


@pytest.mark.parametrize("nx,nv,vs", [(16, 8, 8.0), (32, 32, 8.0), (128, 64, 8.0), (256, 64, 8.0),
                                      (512, 128, 8.0), (1024, 128, 8.0), (8192, 256, 10.0),
                                      (16, 9, 8.0), (20, 12, 5.0), (64, 512, 8.0)])
def test_mesh_matches_reference(gold, nx, nv, vs):
    """build_mesh reproduces the reference grid bit for bit (mesh.py:197-236)."""
    d = gold("mesh")
    k = f"{nx}_{nv}_{vs:g}"
    m = pk.build_mesh(pk.MeshSpec(nx=nx, nvx=nv, v_star=vs))
    g = m.vgrid
    assert np.array_equal(g.vx, d["vx_" + k])
    assert np.array_equal(g.M.reshape(-1), d["M_" + k])
    assert [m.dx, g.dvx, g.dv3, g.m0, g.m2] == list(d["s_" + k])
    assert g.M.shape == (nv, 1, 1) and g.xi.shape == (nv, 1, 1)


def test_mesh_validation():
    with pytest.raises(pk.MeshTooSmall):
        pk.build_mesh(pk.MeshSpec(nx=6, nvx=8))
    with pytest.raises(pk.MeshTooSmall):
        pk.build_mesh(pk.MeshSpec(nx=16, nvx=3))
    with pytest.raises(pk.MeshTooSmall):  # 3V grids follow the reference's >= 4 rule
        pk.build_mesh(pk.MeshSpec(nx=16, nvx=8, nvy=2, nvz=4))
    m3 = pk.build_mesh(pk.MeshSpec(nx=16, nvx=8, nvy=4, nvz=4))
    assert m3.vgrid.shape == (8, 4, 4) and (m3.nv, m3.nvx, m3.nvyz) == (128, 8, 16)
    with pytest.raises(ValueError):
        pk.build_mesh(pk.MeshSpec(nx=16, nvx=8, v_star=-1.0))


def test_bracket_folded_pairwise():
    m = pk.build_mesh(pk.MeshSpec(nx=8, nvx=32))
    rng = np.random.default_rng(3)
    q = rng.standard_normal((8, 32, 1, 1))
    assert np.array_equal(m.bracket_x(q), O.vsum(q.reshape(8, 32), m.vgrid.dv3))
    # odd-in-xi integrands vanish exactly (mesh.py:10-12)
    assert not m.bracket_x(m.xi_M[None] * np.ones((8, 1, 1, 1))).any()


def test_config_inputs_match_reference(gold):
    d = gold("kinetic")
    c = configs.cfg1()
    assert np.array_equal(c.rho, d["c1_rho0"])
    assert np.array_equal(c.g.reshape(128, 64), d["c1_g0"])
    assert c.rho_bar == float(d["c1_rb"])
    p = gold("parareal")
    c2 = configs.cfg2()
    assert np.array_equal(c2.rho, p["c2_rho0"]) and c2.rho_bar == float(p["c2_rb"])


def test_cfg3_cfg4_inputs():
    c3 = configs.cfg3()
    assert c3.rho.shape == (512,) and abs(c3.g).max() < 1e-17  # f = rho M: g = 0
    prof = c3.eps
    assert prof.iface.min() == 1e-3 and 0.5 < prof.iface.max() < 0.5011
    c4 = configs.cfg4(nx=256, nv=32)  # the seeded recipe at reduced size
    rng = np.random.default_rng(0)
    a = rng.uniform(0, 0.05, 8)
    assert abs(c4.rho.mean() - 1.0) < a.sum()


@pytest.mark.parametrize("eps", [1.0, 0.5, 0.1, 1e-2, 1e-4, 1e-6])
@pytest.mark.parametrize("e_max", [0.0, 0.37])
def test_stable_dt_matches_oracle(eps, e_max):
    m = pk.build_mesh(pk.MeshSpec(nx=64, nvx=32))
    g = O.make_grid(64, 32)
    dt = pk.stable_dt(m, eps, e_max=e_max)
    assert dt == O.stable_dt_scalar(g, eps, e_max)
    pk.KineticStepParams(eps=eps, dt=dt).check(dt, m)


def test_stable_dt_eps_profile_is_min():
    m = pk.build_mesh(pk.MeshSpec(nx=64, nvx=32))
    prof = pk.EpsProfile.from_function(configs.eps_bump, m)
    assert pk.stable_dt(m, prof) == min(pk.stable_dt(m, e) for e in prof.distinct())


def test_step_checks():
    m = pk.build_mesh(pk.MeshSpec(nx=32, nvx=32))
    parabolic = m.dx**2 / (2.0 * m.vgrid.m2)
    with pytest.raises(pk.StabilityViolation):
        pk.KineticStepParams(eps=0.5, dt=2.0 * parabolic).check(2.0 * parabolic, m)
    dt_par = 0.9 * parabolic
    pk.KineticStepParams(eps=1e-4, dt=dt_par).check(dt_par, m)
    with pytest.raises(pk.StabilityViolation):
        pk.KineticStepParams(eps=0.1, dt=dt_par).check(dt_par, m)
    with pytest.raises(ValueError):
        pk.KineticStepParams(eps=0.0, dt=1e-3)
    fp = pk.FluidStepParams.default(m)
    with pytest.raises(pk.StabilityViolation):
        fp.check(3.0 * fp.dt, m)


def test_baseline_dt_values_are_infeasible():
    """BASELINE's cfg2 dt choices violate the reference's guards."""
    c = configs.cfg2()
    with pytest.raises(pk.StabilityViolation):
        pk.KineticStepParams(eps=1e-2, dt=1e-4).check(1e-4, c.mesh)
    with pytest.raises(pk.StabilityViolation):
        pk.FluidStepParams.default(c.mesh).check(1e-2, c.mesh)


@pytest.mark.parametrize("t0,t1,dt", [(0.0, 0.2, 1e-3), (0.0, 0.0, 1e-3), (0.1, 0.35, 0.07),
                                      (0.0, 1.0 / 32, 2.766874e-5), (0.3, 0.6, 0.1)])
def test_substep_sizes(t0, t1, dt):
    assert substep_sizes(t0, t1, dt) == O.schedule(t0, t1, dt)


def test_substep_rejects_backwards():
    with pytest.raises(ValueError):
        substep_sizes(1.0, 0.5, 0.1)


def test_relaxation_coefficients_branches():
    k1, k2 = relaxation_coefficients(0.01, 1e-8)
    assert k1 == 0.0 and k2 == 1e-8
    k1, k2 = relaxation_coefficients(0.01, 1e6)
    assert k1 == pytest.approx(1.0, abs=1e-13) and k2 == pytest.approx(0.01 / 1e6, rel=1e-7)
    assert (k1, k2) == O.kappas(0.01, 1e6)


def test_make_phase_constants():
    m = pk.build_mesh(pk.MeshSpec(nx=32, nvx=16))
    prof = pk.EpsProfile.from_function(configs.eps_bump, m)
    ph = make_phase(m, [0.5, prof], [1e-4, 2e-5], [7, 3])
    assert list(ph.nsteps) == [7, 3]
    assert (ph.k1[0] == O.kappas(1e-4, 0.5)[0]).all()
    assert ph.cmac[0, 0] == 1e-4 / (0.5 * m.dx)
    for i in (0, 5, 16, 31):
        e = float(prof.iface[i])
        assert ph.k2[1, i] == O.kappas(2e-5, e)[1] and ph.cmac[1, i] == 2e-5 / (e * m.dx)
    assert ph.cflu[1] == m.vgrid.m2 * (2e-5 / m.dx)


def test_error_mapping():
    for code, cls in [(1, pk.SolvabilityViolation), (2, pk.NonFiniteState),
                      (3, pk.StabilityViolation), (4, pk.MeshTooSmall), (5, ValueError),
                      (7, ValueError), (8, ValueError), (6, errors.NativeError)]:
        with pytest.raises(cls):
            errors.raise_for(code, "x")
    errors.raise_for(0)
    assert issubclass(pk.SolvabilityViolation, pk.SimulationError)


def test_cost_model():
    """parareal.py:438-452 worked example (acceptance criterion 12)."""
    t, k_opt, beats = pk.predict_cost(pk.PerfModel(t_hmm=10.0, t_fluid=1.0, t_lift=1.0,
                                                   n_workers=4, ng=10, k=2))
    assert t == 81.0 and beats
    assert k_opt == math.ceil((10 * 10.0 - 1.0) / (10 * ((1 + 10 + 1) / 4 + 1)))
    with pytest.raises(ValueError):
        pk.PerfModel(t_hmm=-1.0, t_fluid=1.0, t_lift=1.0, n_workers=1, ng=1, k=1)


def test_parareal_config_validation():
    with pytest.raises(ValueError):
        pk.PararealConfig(eps=0.5, t_final=1.0, ng=0)
    with pytest.raises(ValueError):
        pk.PararealConfig(eps=0.5, t_final=1.0, ng=4, tol=0.0)
    cfg = pk.PararealConfig(eps=0.5, t_final=0.3, ng=6)
    assert np.array_equal(cfg.boundaries, np.linspace(0.0, 0.3, 7))


def test_thresholds_and_labels():
    with pytest.raises(ValueError):
        pk.Thresholds(0.0, 1.0)
    lab = pk.DomainLabels.from_cells(np.array([0, 1, 0, 0, 0, 0, 0, 1], dtype=bool))
    assert list(lab.kinetic_ifaces) == [True, True, False, False, False, False, True, True]
    assert lab.kinetic_fraction == 0.25


def test_no_gpu_means_loud_failure():
    """The product has no CPU fallback: without CUDA the device engine raises."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    m = pk.build_mesh(pk.MeshSpec(nx=16, nvx=8))
    with pytest.raises(errors.NativeError):
        pk.solve_field(np.ones(16), 1.0, m)
