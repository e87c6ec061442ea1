"""Generate the golden vectors that pin the oracle to the REAL reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``parakin`` from /root/reference/pkg/src (read-only), builds 1V
meshes by bypassing ``MeshSpec.validate``'s nvy/nvz >= 4 check,
runs the reference through its own public functions, and writes
``tests/golden/*.npz``.  Large arrays are stored as sha256 digests of their
bytes plus a few summary values; everything else is stored verbatim.

The initial-data recipes (``f_*`` below) are the BASELINE.json config formulas
evaluated with the reference's own mesh and bracket (experiment.py:64-85
decomposition).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import parakin.mesh as pm  # noqa: E402
from parakin.adaptation import Thresholds  # noqa: E402
from parakin.fluid import FluidStepParams, fluid_propagate  # noqa: E402
from parakin.hybrid import HybridOptions, HybridState, hybrid_propagate  # noqa: E402
from parakin.kinetic import KineticStepParams, kinetic_propagate, kinetic_step  # noqa: E402
from parakin.lifting import lift  # noqa: E402
from parakin.mesh import MacroState, MeshSpec, MicroState, build_mesh  # noqa: E402
from parakin.parareal import PararealConfig, lift_restart_reference, run  # noqa: E402
from parakin.poisson import solve_field  # noqa: E402
from parakin.errors import SolvabilityViolation  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def mesh1v(nx, nv, v_star=8.0, x_star=2.0 * np.pi):
    """build_mesh with nvy = nvz = 1 (validate bypassed)."""
    spec = MeshSpec(nx=nx, nvx=nv, nvy=1, nvz=1, x_star=x_star, v_star=v_star)
    orig = MeshSpec.validate
    MeshSpec.validate = lambda self: None
    try:
        return build_mesh(spec)
    finally:
        MeshSpec.validate = orig


def digest(a) -> str:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return hashlib.sha256(a.tobytes()).hexdigest()


def g2(g):
    return np.ascontiguousarray(g.reshape(g.shape[0], -1))


def decompose(mesh, f_of_x):
    """experiment.py:64-85 applied to an arbitrary f(x, v)."""
    grid = mesh.vgrid
    f_c = f_of_x(mesh.x_centers)[:, :, None, None]
    rho = mesh.bracket_x(f_c)
    f_if = f_of_x(mesh.x_interfaces)[:, :, None, None]
    rho_if = mesh.bracket_x(f_if)
    g0 = f_if - rho_if[:, None, None, None] * grid.M
    rho_bar = float(rho.sum() * mesh.dx / mesh.x_star)
    return rho, g0, rho_bar


# --- BASELINE.json initial data (builder-chosen conventions) --

def f_cfg1(mesh):
    M = mesh.vgrid.M[:, 0, 0]
    return lambda x: (1.0 + 0.5 * np.cos(x))[:, None] * M[None, :]


def f_cfg2(mesh, eps):
    M = mesh.vgrid.M[:, 0, 0]
    vM = mesh.vgrid.vx * M
    return lambda x: ((1.0 + 0.3 * np.cos(x) + 0.1 * np.sin(2.0 * x))[:, None] * M[None, :]
                      + (1e-3 * eps) * np.cos(x)[:, None] * vM[None, :])


def f_cfg3(mesh):
    M = mesh.vgrid.M[:, 0, 0]
    return lambda x: (1.0 + 0.5 * np.cos(x))[:, None] * M[None, :]


def cfg5_instance(s):
    rng = np.random.default_rng(s)
    a = rng.uniform(0.0, 0.1, 4)
    ph = rng.uniform(0.0, 2.0 * np.pi, 4)
    eps = float(10.0 ** rng.uniform(-4.0, 0.0))
    return a, ph, eps


def f_cfg5(mesh, s):
    a, ph, _ = cfg5_instance(s)
    M = mesh.vgrid.M[:, 0, 0]
    vx = mesh.vgrid.vx

    def f(x):
        rho_in = np.ones_like(x)
        for k in range(4):
            rho_in = rho_in + a[k] * np.cos((k + 1) * x + ph[k])
        return (rho_in[:, None] * M[None, :]) * (1.0 + 0.01 * vx[None, :] * np.cos(x)[:, None])
    return f


def f_paper(mesh):
    """experiment.py:5 reference data f = M xi^4 (1 + 0.9 cos x) (1V)."""
    M = mesh.vgrid.M[:, 0, 0]
    w = mesh.vgrid.vx**4 * M
    return lambda x: w[None, :] * (1.0 + 0.9 * np.cos(2.0 * np.pi * x / mesh.x_star))[:, None]


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def gen_mesh():
    out = {}
    for nx, nv, vs in [(16, 8, 8.0), (32, 32, 8.0), (128, 64, 8.0), (256, 64, 8.0),
                       (512, 128, 8.0), (1024, 128, 8.0), (8192, 256, 10.0),
                       (16, 9, 8.0), (20, 12, 5.0), (64, 512, 8.0)]:
        m = mesh1v(nx, nv, vs)
        k = f"{nx}_{nv}_{vs:g}"
        out[f"vx_{k}"] = m.vgrid.vx
        out[f"M_{k}"] = m.vgrid.M[:, 0, 0]
        out[f"s_{k}"] = np.array([m.dx, m.vgrid.dvx, m.vgrid.dv3, m.vgrid.m0, m.vgrid.m2])
    save("mesh", **out)


def gen_field():
    out = {}
    rng = np.random.default_rng(7)
    for nx in (16, 128, 256, 1000, 8192):
        m = mesh1v(nx, 8)
        d = rng.standard_normal(nx)
        rho = 2.0 + 0.5 * (d - d.mean())
        out[f"rho_{nx}"] = rho
        out[f"E_{nx}"] = solve_field(rho, 2.0, m)
    # guard: a clearly incompatible density raises
    m = mesh1v(64, 8)
    bad = np.full(64, 2.0)
    bad[3] += 1e-3
    try:
        solve_field(bad, 2.0, m)
        out["guard_raised"] = np.array(False)
    except SolvabilityViolation:
        out["guard_raised"] = np.array(True)
    out["guard_rho"] = bad
    save("field", **out)


def gen_kinetic():
    out = {}
    # cfg1 in full: 128x64, eps=1, dt=1e-3, 200 steps
    m = mesh1v(128, 64)
    rho, g0, rb = decompose(m, f_cfg1(m))
    out["c1_rho0"], out["c1_g0"], out["c1_rb"] = rho, g2(g0), np.array(rb)
    E0 = solve_field(rho, rb, m)
    p = KineticStepParams(eps=1.0, dt=1e-3)
    mac, mic = kinetic_propagate((MacroState(rho, E0, 0.0), MicroState(g0)), 0.2, p, m, rb)
    out["c1_rho"], out["c1_E"], out["c1_g"] = mac.rho, mac.E, g2(mic.g)
    # paper data at 32x32, two eps, auto dt with a clipped remainder
    m = mesh1v(32, 32)
    rho, g0, rb = decompose(m, f_paper(m))
    out["p_rho0"], out["p_g0"], out["p_rb"] = rho, g2(g0), np.array(rb)
    E0 = solve_field(rho, rb, m)
    for eps in (0.5, 1e-4):
        p = KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
        t_end = 37.5 * p.dt
        mac, mic = kinetic_propagate((MacroState(rho, E0, 0.0), MicroState(g0)), t_end, p, m, rb)
        k = f"p_{eps:g}"
        out[k + "_dt"] = np.array([p.dt, t_end])
        out[k + "_rho"], out[k + "_E"], out[k + "_g"] = mac.rho, mac.E, g2(mic.g)
    # cfg5 instances at full size: 5 kinetic_step calls at the default dt
    m = mesh1v(1024, 128)
    for s in (0, 1):
        rho, g0, rb = decompose(m, f_cfg5(m, s))
        _, _, eps = cfg5_instance(s)
        E0 = solve_field(rho, rb, m)
        p = KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
        st = (MacroState(rho, E0, 0.0), MicroState(g0))
        for _ in range(5):
            st = kinetic_step(st, p, m, rb)
        k = f"c5_{s}"
        out[k + "_init"] = np.array([digest(rho), digest(g2(g0))])
        out[k + "_rho0"] = rho
        out[k + "_par"] = np.array([rb, eps, p.dt])
        out[k + "_rho"], out[k + "_E"] = st[0].rho, st[0].E
        out[k + "_g"] = np.array(digest(g2(st[1].g)))
    save("kinetic", **out)


HYB_CASES = [
    # name, data, nx, nv, eps, delta0, eta0, opts, steps, field_rtol
    ("p_1e-2_or", "paper", 48, 16, 1e-2, 1e-3, 1e-3, dict(), 200, 1e-2),
    ("p_1e-3_or", "paper", 48, 16, 1e-3, 1e-5, 1e-5, dict(), 200, 1e-2),
    ("p_0.5_or", "paper", 48, 16, 0.5, 1e-2, 1e-2, dict(), 200, 1e-2),
    ("l_1e-3_and", "lift", 48, 16, 1e-3, 1e-2, 1e-2, dict(combine="and"), 200, 1e-2),
    ("l_1e-3_and_zero", "lift", 48, 16, 1e-3, 1e-2, 1e-2,
     dict(combine="and", reinit="zero"), 200, 1e-2),
    ("l_1e-3_and_o1", "lift", 48, 16, 1e-3, 1e-2, 1e-2,
     dict(combine="and", lift_order=1), 200, 1e-2),
    ("l_1e-3_and_ho", "lift", 48, 16, 1e-3, 1e-2, 1e-2,
     dict(combine="and", time_elim="higher_order"), 200, 1e-2),
    ("l_1e-3_and_th3", "lift", 48, 16, 1e-3, 1e-3, 1e-3, dict(combine="and"), 200, 1e-2),
    ("l_0.1_or", "lift", 48, 16, 0.1, 1e-3, 1e-3, dict(), 200, 1e-2),
    ("l_0.5_and", "lift", 48, 16, 0.5, 1e-2, 1e-2, dict(combine="and"), 200, 1e-2),
    ("p_scaled", "paper", 48, 16, 1e-2, 1e-7, 1e-3, dict(scale_remainder=True), 200, 1e-2),
    ("p_1e-4_guard", "paper", 32, 32, 1e-4, 1e-5, 1e-5, dict(), 300, 1e-5),
    ("p_1e-2_guard", "paper", 32, 32, 1e-2, 1e-3, 1e-3, dict(), 200, 1e-5),
    ("p_1e-4_big", "paper", 64, 32, 1e-4, 1e-5, 1e-5, dict(), 300, 1e-2),
    ("loose", "paper", 24, 8, 0.5, 1e9, 1e9, dict(), 50, 1e-5),
]


def hyb_input(data, nx, nv, eps):
    m = mesh1v(nx, nv)
    if data == "paper":
        rho, g0, rb = decompose(m, f_paper(m))
        E0 = solve_field(rho, rb, m)
    else:
        rho, _, rb = decompose(m, f_cfg3(m))
        E0 = solve_field(rho, rb, m)
        g0 = lift(rho, E0, eps, m, rho_bar=rb).g
    return m, rho, g0, rb, E0


def gen_hybrid():
    out = {}
    for name, data, nx, nv, eps, d0, e0, kw, nsteps, rtol in HYB_CASES:
        m, rho, g0, rb, E0 = hyb_input(data, nx, nv, eps)
        p = KineticStepParams.default(m, eps, e_max=float(np.abs(E0).max()))
        opts = HybridOptions(adaptation=True, **kw)
        th = Thresholds(d0, e0)
        st = HybridState.initial(MacroState(rho, E0, 0.0), MicroState(g0), m)
        kc_trace = []
        t_end = (nsteps + 0.5) * p.dt
        k = "h_" + name
        out[k + "_in"] = np.concatenate([rho, g2(g0).ravel(), [rb, p.dt, t_end]])
        try:
            st = hybrid_propagate(st, t_end, p, th, opts, m, rb, field_rtol=rtol,
                                  trace=lambda s: kc_trace.append(s.labels.kinetic_cells.copy()))
        except SolvabilityViolation:
            out[k + "_raised"] = np.array(len(kc_trace))
            print(name, "raised SolvabilityViolation after", len(kc_trace), "steps")
            continue
        out[k + "_rho"], out[k + "_E"], out[k + "_g"] = st.macro.rho, st.macro.E, g2(st.micro.g)
        out[k + "_kc"], out[k + "_ki"] = st.labels.kinetic_cells, st.labels.kinetic_ifaces
        out[k + "_Eprev"] = st.E_prev
        out[k + "_trace"] = np.array(kc_trace)
    save("hybrid", **out)


def gen_lift():
    out = {}
    m = mesh1v(64, 32)
    rho, g0, rb = decompose(m, f_paper(m))
    E = solve_field(rho, rb, m)
    E_prev = E * (1.0 + 1e-3 * np.sin(m.x_interfaces))
    for eps in (0.5, 1e-3):
        for order in (1, 2):
            for te in ("leading", "higher_order"):
                for proj in (True, False):
                    g = lift(rho, E, eps, m, order=order, time_elim=te, rho_bar=rb,
                             dE_dt=(E - E_prev) / 1e-4, project=proj).g
                    out[f"l_{eps:g}_{order}_{te}_{int(proj)}"] = g2(g)
    out["rho"], out["E"], out["E_prev"], out["rb"] = rho, E, E_prev, np.array(rb)
    save("lift", **out)


def gen_fluid():
    out = {}
    m = mesh1v(256, 64)
    rho, _, rb = decompose(m, f_cfg2(m, 1e-2))
    fp = FluidStepParams.default(m)
    st = fluid_propagate(MacroState(rho, np.zeros(256), 0.0), 0.5 / 16, fp, m, rb)
    out["rho0"], out["rb"], out["rho"], out["E"] = rho, np.array(rb), st.rho, st.E
    out["dt"] = np.array(fp.dt)
    save("fluid", **out)


PAR_CASES = [
    ("off_0.5", 32, 16, 0.5, False, 6, 0.3, 12, 1e-10, 1e-5, 1e-5),
    ("off_1e-4", 32, 16, 1e-4, False, 6, 0.3, 12, 1e-10, 1e-5, 1e-5),
    ("on_1e-4", 32, 16, 1e-4, True, 6, 0.3, 12, 1e-10, 1e-5, 1e-5),
    ("on_1e-2", 32, 16, 1e-2, True, 5, 0.2, 8, 1e-10, 1e-3, 1e-3),
]


def gen_parareal(full_cfg2=True):
    out = {}
    for name, nx, nv, eps, adapt, ng, T, kmax, tol, d0, e0 in PAR_CASES:
        m = mesh1v(nx, nv)
        rho, g0, rb = decompose(m, f_paper(m))
        cfg = PararealConfig(eps=eps, t_final=T, ng=ng, k_max=kmax, tol=tol, workers=1,
                             thresholds=Thresholds(d0, e0),
                             options=HybridOptions(adaptation=adapt))
        try:
            res = run(cfg, rho, g2(g0).reshape(g0.shape), m, rb)
        except SolvabilityViolation:
            out[f"p_{name}_raised"] = np.array(True)
            continue
        k = f"p_{name}"
        out[k + "_rows"] = np.stack(res.ledger.rho)
        out[k + "_err"] = np.array(res.ledger.err)
        out[k + "_frac"] = res.kinetic_fraction
        out[k + "_meta"] = np.array([res.iterations, res.status == "converged"])
        if not adapt:
            out[k + "_chain"] = lift_restart_reference(cfg, rho, g0, m, rb)
    if full_cfg2:
        m = mesh1v(256, 64)
        eps = 1e-2
        rho, g0, rb = decompose(m, f_cfg2(m, eps))
        cfg = PararealConfig(eps=eps, t_final=0.5, ng=16, k_max=5, tol=1e-10, workers=1,
                             options=HybridOptions(adaptation=False))
        tic = time.perf_counter()
        res = run(cfg, rho, g0, m, rb)
        wall = time.perf_counter() - tic
        out["c2_rho0"], out["c2_rb"] = rho, np.array(rb)
        out["c2_g0"] = np.array(digest(g2(g0)))
        out["c2_rows"] = np.stack(res.ledger.rho)
        out["c2_err"] = np.array(res.ledger.err)
        out["c2_meta"] = np.array([res.iterations, res.status == "converged", wall])
        print(f"cfg2 reference run: {res.status} in {res.iterations} iterations, {wall:.1f} s")
    save("parareal", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["mesh", "field", "kinetic", "hybrid", "lift", "fluid", "parareal"]
    for w in which:
        globals()["gen_" + w]()
