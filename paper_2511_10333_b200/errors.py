"""Error taxonomy of the EDGC surface.

Class names and base classes match the reference (pkg/src/edgc/errors.py:4-29)
so ``except`` clauses written against the reference keep working; device-side
status words from libedgc_b200.so are mapped onto these in ``_lib.py``.
"""

__all__ = ["EdgcError", "DegenerateInputError", "TraceFormatError", "CalibrationError",
           "CompressionInfeasibleError", "DivergenceError", "ConfigError"]


class EdgcError(Exception):
    pass


class DegenerateInputError(EdgcError, ValueError):
    """Sample without spread: zero variance / zero range / a window with no records."""


class TraceFormatError(EdgcError, ValueError):
    """EDGT trace bytes do not parse."""


class CalibrationError(EdgcError, ValueError):
    """The comm-time fit is underdetermined or non-positive."""


class CompressionInfeasibleError(EdgcError, RuntimeError):
    """Even rank 1 costs more than sending the raw gradient."""


class DivergenceError(EdgcError, RuntimeError):
    """A loss or gradient went non-finite."""


class ConfigError(EdgcError, ValueError):
    """A run configuration failed schema validation."""
