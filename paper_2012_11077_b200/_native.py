"""ctypes binding of the C ABI (include/uwbvital_b200.h).

Loads ``lib/libuwbvital_b200.so`` built in-tree by ``build.py``. There is no
Python or CPU fallback: if the library is missing the import fails, and every
compute call returns ``UWB_CUDA_ERROR`` (raised as :class:`CudaError`) when no
CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libuwbvital_b200.so")
DROPIN_PATH = os.path.join(HERE, "lib", "libuwbvital.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing; build it with `python __graft_entry__.py` "
                      "(the package has no CPU fallback)")

lib = C.CDLL(LIB_PATH)

# ---------------------------------------------------------------- status ---
UWB_OK = 0
UWB_DIMENSION_ERROR = 1
UWB_INPUT_ERROR = 2
UWB_PARAMETER_ERROR = 3
UWB_BOUNDS_ERROR = 4
UWB_CONFIGURATION_ERROR = 5
UWB_CUDA_ERROR = 6
UWB_CAPACITY_ERROR = 7
UWB_INVALID_ARGUMENT = 8
UWB_FORMAT_ERROR = 9

UWB_F32 = 0
UWB_F64 = 1
UWB_NAIVE = 0
UWB_INTEGRAL = 1
UWB_SAT_GLOBAL = 0
UWB_SAT_SLAB = 1
UWB_SAT_TILE = 2


class uwb_cfar_params(C.Structure):
    _fields_ = [("guard_rows", C.c_int32), ("guard_cols", C.c_int32),
                ("background_rows", C.c_int32), ("background_cols", C.c_int32),
                ("pfa", C.c_double)]


class uwb_detection(C.Structure):
    _fields_ = [("row", C.c_uint64), ("col", C.c_uint64), ("value", C.c_double),
                ("threshold", C.c_double)]


class uwb_pipeline_config(C.Structure):
    _fields_ = [("mean_filter_window", C.c_uint64), ("fft_length", C.c_uint64),
                ("band_low_hz", C.c_double), ("band_high_hz", C.c_double),
                ("cfar", uwb_cfar_params), ("backend", C.c_int32),
                ("mean_filter_mode", C.c_int32), ("normalization_epsilon", C.c_double)]


class uwb_map_batch(C.Structure):
    _fields_ = [("maps", C.c_void_p), ("dtype", C.c_int32), ("reserved", C.c_int32),
                ("n_maps", C.c_uint64), ("rows", C.c_uint64), ("cols", C.c_uint64),
                ("ld", C.c_uint64), ("map_stride", C.c_uint64)]


class uwb_row_window(C.Structure):
    _fields_ = [("global_rows", C.c_uint64), ("buf_row0", C.c_uint64), ("row_begin", C.c_uint64),
                ("row_end", C.c_uint64), ("col_bands", C.c_uint64)]


class uwb_rfrm_info(C.Structure):
    _fields_ = [("m_samples", C.c_uint32), ("n_traces", C.c_uint32), ("fast_rate", C.c_double),
                ("prf", C.c_double), ("payload_offset", C.c_uint64), ("payload_bytes", C.c_uint64)]


class uwb_cfar_outputs(C.Structure):
    _fields_ = [("mask_bits", C.c_void_p), ("words_per_row", C.c_uint64),
                ("mask_map_stride", C.c_uint64), ("mask_u8", C.c_void_p),
                ("thresholds", C.c_void_p), ("dets", C.c_void_p), ("det_capacity", C.c_uint64),
                ("det_counts", C.c_void_p), ("first_bad", C.c_void_p),
                ("tie_counts", C.c_void_p), ("ties", C.c_void_p), ("tie_capacity", C.c_uint64),
                ("cert_status", C.c_void_p)]


_P = C.c_void_p
_U64 = C.c_uint64
_D = C.c_double
_S = C.c_int  # uwb_status

# Every symbol the header declares, with its signature. tests/test_abi.py checks
# this table against include/uwbvital_b200.h and the exported symbols.
SIGNATURES = {
    "uwb_last_error": (C.c_char_p, []),
    "uwb_last_error_cell": (None, [_P, _P]),
    "uwb_device_available": (C.c_int, []),
    "uwb_alpha_factor": (_S, [_U64, _D, _P]),
    "uwb_cfar_params_validate": (_S, [_P]),
    "uwb_interior_train_count": (_U64, [_P]),
    "uwb_training_window": (_S, [_P, _U64, _U64, _U64, _U64, _P]),
    "uwb_alpha_table": (_S, [_P, _P, _U64]),
    "uwb_build_sat": (_S, [_P, _U64, _U64, _P]),
    "uwb_cfar2d": (_S, [C.c_int, _P, _U64, _U64, _P, _P, _P, _P, _U64, _P]),
    "uwb_remove_dc": (_S, [_P, _U64, _U64, _P]),
    "uwb_detrend_linear": (_S, [_P, _U64, _U64, _P]),
    "uwb_mean_filter_slow": (_S, [_P, _U64, _U64, _U64, _P]),
    "uwb_subtract_slow_time_mean": (_S, [_P, _U64, _U64, _P]),
    "uwb_normalize_slow": (_S, [_P, _U64, _U64, _D, _P]),
    "uwb_slow_time_spectrum": (_S, [_P, _U64, _U64, _D, _D, _U64, _P, _P, _P]),
    "uwb_band_select": (_S, [_P, _U64, _U64, _P, _D, _D, _P, _P, _P, _P]),
    "uwb_detect": (_S, [_P, _U64, _U64, _D, _D, _P, _U64, _P, _P, _P, _P, _P, _P, _P, _U64, _P]),
    "uwb_dev_cfar2d_workspace": (_U64, [_P, _P, C.c_int32, _U64, _U64]),
    "uwb_dev_cfar2d": (_S, [_P, _P, _P, C.c_int32, _U64, _P, _P, _U64, C.c_uint32, _P]),
    "uwb_dev_cfar2d_window_workspace": (_U64, [_P, _P, _P, _U64, _U64]),
    "uwb_dev_cfar2d_window": (_S, [_P, _P, _P, _P, _U64, _P, _P, _U64, C.c_uint32, _P]),
    "uwb_dev_detect_batch_workspace": (_U64, [_U64, _U64, _U64, _D, _P, _U64]),
    "uwb_dev_detect_batch": (_S, [_P, C.c_int32, _U64, _U64, _U64, _D, _D, _P, _P, _P, _P, _P, _U64, C.c_uint32, _P]),
    "uwb_rfrm_parse": (_S, [_P, _U64, _P]),
    "uwb_dev_rfrm_to_frames": (_S, [_P, _U64, _U64, _U64, C.c_int32, _P, _P, _P]),
    "uwb_dev_build_sat": (_S, [_P, _P, _U64, _U64, _P, _P, _U64, _P]),
    "uwb_dev_build_sat_workspace": (_U64, [_P]),
    "uwb_host_cfar2d_batch": (_S, [_P, _P, C.c_int32, _U64, _P, _P, _U64, _P, _U64]),
    "uwb_kernel_launches": (_U64, []),
    "uwb_dev_phase_ms": (C.c_int32, [_P, C.c_int32]),
    "uwb_dev_phase_ms4": (C.c_int32, [_P, C.c_int32]),
    "uwb_host_alloc": (_P, [_U64]),
    "uwb_host_free": (None, [_P]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def last_error() -> str:
    return (lib.uwb_last_error() or b"").decode()


def last_error_cell() -> tuple[int, int]:
    r, c = C.c_int64(), C.c_int64()
    lib.uwb_last_error_cell(C.byref(r), C.byref(c))
    return r.value, c.value


def device_available() -> bool:
    return bool(lib.uwb_device_available())
