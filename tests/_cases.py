"""Shared test inputs: the same recipes as tests/golden/make_golden.py, built
with the ORACLE's grid (CPU tests) or the product's mesh (GPU tests)."""

import hashlib

import numpy as np


def digest(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return hashlib.sha256(a.tobytes()).hexdigest()


def cdigest(a):
    """digest() with every NaN replaced by numpy's canonical quiet NaN: x86
    and the GPU produce different NaN payloads (tests/golden/make_cfg5_golden.py)."""
    a = np.array(a, dtype=np.float64, copy=True)
    a[np.isnan(a)] = np.nan
    return digest(a)


def f_paper(vx, M, x_star):
    w = vx**4 * M
    return lambda x: w[None, :] * (1.0 + 0.9 * np.cos(2.0 * np.pi * x / x_star))[:, None]


def f_cfg3(M):
    return lambda x: (1.0 + 0.5 * np.cos(x))[:, None] * M[None, :]


def f_cfg1(M):
    return lambda x: (1.0 + 0.5 * np.cos(x))[:, None] * M[None, :]


HYB_CASES = [
    # name, data, nx, nv, eps, delta0, eta0, opts, steps, field_rtol (make_golden.py)
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

PAR_CASES = [
    ("off_0.5", 32, 16, 0.5, False, 6, 0.3, 12, 1e-10, 1e-5, 1e-5),
    ("off_1e-4", 32, 16, 1e-4, False, 6, 0.3, 12, 1e-10, 1e-5, 1e-5),
    ("on_1e-4", 32, 16, 1e-4, True, 6, 0.3, 12, 1e-10, 1e-5, 1e-5),
    ("on_1e-2", 32, 16, 1e-2, True, 5, 0.2, 8, 1e-10, 1e-3, 1e-3),
]
