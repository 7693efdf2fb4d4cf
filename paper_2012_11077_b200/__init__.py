"""B200-native (sm_100a) drop-in for the uwbvital north-star path of arXiv 2012.11077:
front-end preprocessing -> slow-time FFT / band select -> summed-area table ->
2-D CA-CFAR.

The public API mirrors the reference's C++ headers (proj/include/uwbvital/
{sat,cfar,pipeline}.hpp) function for function; see :mod:`.api`. The batched,
device-resident throughput path is :class:`.batch.BatchCfar`. Everything runs
in the CUDA kernels of ``lib/libuwbvital_b200.so``; importing this package
without that library fails, and compute calls without a GPU raise
:class:`.errors.CudaError` (there is no CPU fallback).
"""
from .errors import (BoundsError, CapacityError, ConfigurationError, CudaError, DimensionError, Error,
                     FormatError, GateError, InputError, ParameterError)
from .api import *  # noqa: F401,F403
from .api import __all__ as _api_all
from ._native import device_available, LIB_PATH, DROPIN_PATH

__all__ = list(_api_all) + [
    "Error", "DimensionError", "InputError", "ParameterError", "BoundsError", "ConfigurationError",
    "FormatError", "GateError", "CudaError", "CapacityError", "device_available", "LIB_PATH",
    "DROPIN_PATH",
]
