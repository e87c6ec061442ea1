"""Exception taxonomy of the drop-in (same names and hierarchy as the
reference, errors.py:4-26), plus the mapping from libpk status codes."""


class SimulationError(Exception):
    """Base class for solver failures."""


class MeshTooSmall(SimulationError):
    """Grid has too few cells for the requested operation (stencils need >= 7)."""


class SolvabilityViolation(SimulationError):
    """Density incompatible with the periodic field equation."""


class StabilityViolation(SimulationError):
    """Time step exceeds the stability bound of the scheme."""


class NonFiniteState(SimulationError):
    """A propagated density became non-finite (blow-up)."""


class ConfigError(SimulationError):
    """Invalid or unparsable run configuration."""


class NativeError(RuntimeError):
    """libpk failed (CUDA error, unsupported shape, missing extension)."""


# include/pk.h PK_ERR_* -> exception class
_BY_CODE = {
    1: SolvabilityViolation,
    2: NonFiniteState,
    3: StabilityViolation,
    4: MeshTooSmall,
    5: ValueError,
    6: NativeError,
    7: ValueError,
    8: ValueError,
    9: NativeError,
}

_MESSAGES = {
    1: "density incompatible with periodic field equation (solvability guard)",
    2: "non-finite density (blow-up)",
    3: "time step exceeds the stability bound",
    4: "mesh too small",
    5: "invalid argument",
    6: "CUDA failure",
    7: "reinit must be 'lift' or 'zero'",
    8: "invalid lift order / time_elim",
    9: "unsupported grid shape",
}


def raise_for(code: int, detail: str = "", slice=None, step=None) -> None:
    """Raise the exception class of a libpk status code.  The raised object
    carries ``pk_code`` and, for device-detected errors, the failing batch
    entry ``pk_slice`` and ``pk_step`` (the parareal engine maps the slice to
    its window)."""
    if code == 0:
        return
    cls = _BY_CODE.get(code, NativeError)
    msg = _MESSAGES.get(code, f"libpk error {code}")
    ex = cls(f"{msg}{': ' + detail if detail else ''}")
    ex.pk_code, ex.pk_slice, ex.pk_step = code, slice, step
    raise ex


def code_of(ex: BaseException) -> int:
    """libpk status code of an exception (inverse of raise_for's classes)."""
    c = getattr(ex, "pk_code", None)
    if c:
        return int(c)
    for code, cls in ((1, SolvabilityViolation), (2, NonFiniteState), (3, StabilityViolation),
                      (4, MeshTooSmall), (5, ValueError)):
        if isinstance(ex, cls):
            return code
    return 6
