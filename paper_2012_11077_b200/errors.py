"""Exception taxonomy mirroring proj/include/uwbvital/errors.hpp:9-47.

The C ABI returns a status code (1..5 map one-to-one onto these classes) and the
reference's message text; :func:`raise_for` turns that into the exception the
reference would have thrown.
"""
from __future__ import annotations

from . import _native as N


class Error(RuntimeError):
    """Common base (errors.hpp:10-12)."""


class DimensionError(Error):
    """Empty or shape-incompatible matrix input."""


class InputError(Error):
    """Non-finite or otherwise invalid data values."""

    def __init__(self, message: str, row: int = -1, col: int = -1):
        super().__init__(message)
        self.row = row
        self.col = col


class ParameterError(Error):
    """Scalar parameter outside its domain."""


class BoundsError(Error):
    """Rectangle or index out of range."""


class ConfigurationError(Error):
    """Configuration incompatible with the data it is applied to."""


class FormatError(Error):
    """Violations of an on-disk format."""


class GateError(Error):
    """Internal correctness gate tripped."""


class CudaError(Error):
    """No usable CUDA device or a CUDA failure (there is no CPU fallback)."""


class CapacityError(Error):
    """Detection buffer too small; ``count`` holds the true number."""

    def __init__(self, message: str, count: int = 0):
        super().__init__(message)
        self.count = count


_CLASSES = {
    N.UWB_DIMENSION_ERROR: DimensionError,
    N.UWB_PARAMETER_ERROR: ParameterError,
    N.UWB_BOUNDS_ERROR: BoundsError,
    N.UWB_CONFIGURATION_ERROR: ConfigurationError,
    N.UWB_CUDA_ERROR: CudaError,
    N.UWB_INVALID_ARGUMENT: ValueError,
    N.UWB_FORMAT_ERROR: FormatError,
}


def raise_for(status: int) -> None:
    if status == N.UWB_OK:
        return
    msg = N.last_error()
    if status == N.UWB_INPUT_ERROR:
        r, c = N.last_error_cell()
        raise InputError(msg, r, c)
    if status == N.UWB_CAPACITY_ERROR:
        raise CapacityError(msg)
    raise _CLASSES.get(status, Error)(msg)
