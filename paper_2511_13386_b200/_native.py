"""ctypes binding of libpk.so (include/pk.h).

The shared library is built in-tree by ``build.py`` (nvcc, sm_100a) and loaded
from this package directory.  There is no fallback: if the library is
missing or no CUDA device is present, every solver entry point raises
:class:`~paper_2511_13386_b200.errors.NativeError`.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
# PK_LIB_PATH: load another build of the same ABI (A/B measurements only)
LIB_PATH = os.environ.get("PK_LIB_PATH") or os.path.join(_HERE, "libpk.so")

c_double_p = C.POINTER(C.c_double)
c_int32_p = C.POINTER(C.c_int32)
c_uint8_p = C.POINTER(C.c_uint8)


class PkMesh(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("nv", C.c_int32),
        ("dx", C.c_double), ("dvx", C.c_double), ("dv3", C.c_double), ("m0", C.c_double),
        ("m2", C.c_double), ("x_star", C.c_double), ("v_star", C.c_double),
        ("vx", c_double_p), ("M", c_double_p), ("xi_M", c_double_p), ("w2", c_double_p),
        ("stencil", (C.c_double * 7) * 4), ("stencil_scale", C.c_double * 4),
        ("nvyz", C.c_int32),
    ]


class PkPhase(C.Structure):
    _fields_ = [
        ("nsteps", C.c_void_p), ("dt", C.c_void_p), ("cflu", C.c_void_p),
        ("kappa1", C.c_void_p), ("kappa2", C.c_void_p), ("cmac", C.c_void_p),
        ("cmac_scalar", C.c_void_p),
        ("kappa1_scalar", C.c_void_p),
        ("kappa2_scalar", C.c_void_p),
    ]


class PkHybrid(C.Structure):
    _fields_ = [
        ("adaptation", C.c_int32), ("combine_and", C.c_int32), ("reinit", C.c_int32),
        ("lift_order", C.c_int32), ("time_elim", C.c_int32), ("exact_scan", C.c_int32),
        ("delta0", C.c_double), ("eta0", C.c_double),
        ("rscale", C.c_void_p), ("neg_eps", C.c_void_p), ("eps2", C.c_void_p),
    ]


class PkStatus(C.Structure):
    _fields_ = [("code", C.c_int32), ("slice", C.c_int32), ("step", C.c_int32),
                ("pad", C.c_int32)]


# symbol -> (restype, argtypes); the full C ABI of include/pk.h
SIGNATURES = {
    "pk_version": (C.c_int32, []),
    "pk_debug_profile": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "pk_count_rows": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "pk_create": (C.c_void_p, [C.c_int32, C.POINTER(PkMesh)]),
    "pk_destroy": (None, [C.c_void_p]),
    "pk_last_error": (C.c_char_p, [C.c_void_p]),
    "pk_reserve": (C.c_int32, [C.c_void_p, C.c_int32]),
    "pk_status_read": (C.c_int32, [C.c_void_p, C.POINTER(PkStatus), C.c_int32]),
    "pk_status_read_stream": (C.c_int32, [C.c_void_p, C.POINTER(PkStatus), C.c_int32, C.c_void_p]),
    "pk_fine_last_launch": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int32)]),
    "pk_fine_cancel": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "pk_fine_propagate": (C.c_int32, [
        C.c_void_p, C.c_int32,
        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
        C.c_void_p, C.c_void_p, C.POINTER(PkPhase), C.POINTER(PkHybrid),
        C.c_double, C.c_int32, C.c_void_p]),
    "pk_coarse_chain": (C.c_int32, [
        C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
        C.c_void_p,
        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
        C.c_double, C.c_void_p, C.c_double, C.c_int32, C.c_void_p]),
    "pk_field": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.c_double, C.c_int32, C.c_void_p]),
    "pk_lift": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                            C.c_int32, C.c_void_p, C.c_void_p]),
    "pk_jump": (C.c_int32, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                            C.c_void_p]),
    "pk_maxdiff": (C.c_int32, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p]),
    "pk_status_store": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "pk_remainder": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]),
    "pk_perturbation": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                    C.c_void_p]),
    "pk_labels": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_double,
                              C.c_double, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "pk_diag_qdiv": (C.c_int32, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libpk.so (once).  Raises NativeError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeError(
            f"{path} not found: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
