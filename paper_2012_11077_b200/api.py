"""Python mirror of the reference's public API (proj/include/uwbvital/*.hpp).

Same names, argument meaning, defaults and exception classes as the C++
library; every function is one call into the C ABI, which runs the arithmetic
on the GPU. Host inputs are numpy arrays (``Matrix`` = float64 2-D array,
``Mask`` = uint8 2-D array).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import CapacityError, raise_for

DETECTION_DTYPE = np.dtype([("row", np.uint64), ("col", np.uint64), ("value", np.float64),
                            ("threshold", np.float64)])


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _matrix(m) -> np.ndarray:
    a = np.ascontiguousarray(m, dtype=np.float64)
    if a.ndim != 2:
        if a.size == 0:
            return a.reshape(0, 0)
        raise ValueError("a 2-D matrix is required")
    return a


# ------------------------------------------------------------------ CFAR ---

@dataclass
class CfarParams:
    """cfar.hpp:19-32, with optional per-axis radii (BASELINE config 5).

    ``guard_radius``/``background_radius`` are the reference's square window;
    ``guard_cols``/``background_cols`` default to them.
    """
    guard_radius: int = 4
    background_radius: int = 8
    pfa: float = 1e-3
    guard_cols: int | None = None
    background_cols: int | None = None

    def to_c(self) -> N.uwb_cfar_params:
        gc = self.guard_radius if self.guard_cols is None else self.guard_cols
        bc = self.background_radius if self.background_cols is None else self.background_cols
        return N.uwb_cfar_params(int(self.guard_radius), int(gc), int(self.background_radius), int(bc),
                                 float(self.pfa))

    def validate(self) -> None:
        p = self.to_c()
        raise_for(N.lib.uwb_cfar_params_validate(C.byref(p)))

    def interior_train_count(self) -> int:
        p = self.to_c()
        return int(N.lib.uwb_interior_train_count(C.byref(p)))

    def alpha_table(self) -> np.ndarray:
        """alpha[n] for n = 0..interior_train_count (AlphaTable, cfar.cpp:65-79)."""
        p = self.to_c()
        out = np.zeros(self.interior_train_count() + 1)
        raise_for(N.lib.uwb_alpha_table(C.byref(p), _ptr(out), C.c_uint64(out.size)))
        return out


@dataclass
class CellRect:
    r0: int
    r1: int
    c0: int
    c1: int

    def area(self) -> int:
        return (self.r1 - self.r0 + 1) * (self.c1 - self.c0 + 1)


@dataclass
class TrainingWindow:
    outer: CellRect
    guard: CellRect
    n_train: int


@dataclass
class DetectionResult:
    mask: np.ndarray           # uint8 rows x cols
    threshold_map: np.ndarray  # float64 rows x cols
    detections: np.ndarray     # DETECTION_DTYPE, value desc, row asc, col asc


def alpha_factor(n_train: int, pfa: float) -> float:
    out = C.c_double()
    raise_for(N.lib.uwb_alpha_factor(C.c_uint64(n_train), C.c_double(pfa), C.byref(out)))
    return out.value


def training_window(params: CfarParams, row: int, col: int, rows: int, cols: int) -> TrainingWindow:
    p = params.to_c()
    out = (C.c_uint64 * 9)()
    raise_for(N.lib.uwb_training_window(C.byref(p), C.c_uint64(row), C.c_uint64(col),
                                        C.c_uint64(rows), C.c_uint64(cols), out))
    o = [int(v) for v in out]
    return TrainingWindow(CellRect(*o[0:4]), CellRect(*o[4:8]), o[8])


def _cfar(backend: int, power_map, params: CfarParams) -> DetectionResult:
    m = _matrix(power_map)
    rows, cols = m.shape
    mask = np.zeros((rows, cols), np.uint8)
    thr = np.zeros((rows, cols), np.float64)
    p = params.to_c()
    cap = max(1, min(rows * cols, 4096))
    while True:
        dets = np.zeros(cap, DETECTION_DTYPE)
        n = C.c_uint64()
        st = N.lib.uwb_cfar2d(backend, _ptr(m), C.c_uint64(rows), C.c_uint64(cols), C.byref(p),
                              _ptr(mask), _ptr(thr), _ptr(dets), C.c_uint64(cap), C.byref(n))
        if st == N.UWB_CAPACITY_ERROR:
            cap = int(n.value)
            continue
        raise_for(st)
        return DetectionResult(mask, thr, dets[: n.value].copy())


def cfar2d_naive(power_map, params: CfarParams, threads: int = 1) -> DetectionResult:
    """cfar.hpp:77-78 (explicit ring sums; bit-identical to the reference naive backend)."""
    return _cfar(N.UWB_NAIVE, power_map, params)


def cfar2d_integral(power_map, params: CfarParams, threads: int = 1) -> DetectionResult:
    """cfar.hpp:83-84 (exact SAT + four-tap sums; bit-identical to the reference)."""
    return _cfar(N.UWB_INTEGRAL, power_map, params)


# ------------------------------------------------------------------- SAT ---

class SummedAreaTable:
    """sat.hpp:16-46. ``table`` is the (M+1)x(N+1) zero-padded fp64 table."""

    def __init__(self, rows: int, cols: int, table: np.ndarray):
        self._rows, self._cols, self._table = rows, cols, table

    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    def table(self) -> np.ndarray:
        return self._table

    def region_sum_unchecked(self, r0, r1, c0, c1) -> float:
        t = self._table
        return float((t[r0, c0] + t[r1 + 1, c1 + 1]) - (t[r0, c1 + 1] + t[r1 + 1, c0]))

    def region_sum(self, r0, r1, c0, c1) -> float:
        from .errors import BoundsError
        if r0 > r1 or c0 > c1 or r1 >= self._rows or c1 >= self._cols:
            raise BoundsError(f"region_sum: invalid rectangle [{r0}..{r1}] x [{c0}..{c1}] on "
                              f"{self._rows}x{self._cols} table")
        return self.region_sum_unchecked(r0, r1, c0, c1)


def build_sat(source) -> SummedAreaTable:
    m = _matrix(source)
    rows, cols = m.shape
    table = np.zeros((rows + 1, cols + 1), np.float64)
    raise_for(N.lib.uwb_build_sat(_ptr(m), C.c_uint64(rows), C.c_uint64(cols), _ptr(table)))
    return SummedAreaTable(rows, cols, table)


# -------------------------------------------------------------- pipeline ---

@dataclass
class RadarFrame:
    """frame.hpp:10-21."""
    data: np.ndarray
    fast_rate: float = 39e9
    prf: float = 68.6

    def samples(self) -> int:
        return int(np.shape(self.data)[0])

    def traces(self) -> int:
        return int(np.shape(self.data)[1])


@dataclass
class PipelineConfig:
    """pipeline.hpp:18-30."""
    mean_filter_window: int = 5
    fft_length: int = 0
    band_low_hz: float = 0.3
    band_high_hz: float = 0.8
    cfar: CfarParams = field(default_factory=CfarParams)
    backend: str = "integral"          # or "naive"
    normalization_epsilon: float = 1e-12
    mean_filter_mode: str = "smoothing"  # or "subtract_mean"

    def effective_fft_length(self, n_traces: int) -> int:
        if self.fft_length:
            return int(self.fft_length)
        p = 1
        while p < n_traces:
            p <<= 1
        return p

    def to_c(self) -> N.uwb_pipeline_config:
        return N.uwb_pipeline_config(
            int(self.mean_filter_window), int(self.fft_length), float(self.band_low_hz),
            float(self.band_high_hz), self.cfar.to_c(),
            N.UWB_NAIVE if self.backend == "naive" else N.UWB_INTEGRAL,
            0 if self.mean_filter_mode == "smoothing" else 1, float(self.normalization_epsilon))


@dataclass
class RangeFrequencyMap:
    power: np.ndarray
    freq_axis: np.ndarray
    range_axis: np.ndarray


@dataclass
class DetectOutput:
    band_map: RangeFrequencyMap
    detections: DetectionResult


def _frame_op(fn, frame: RadarFrame, *extra) -> RadarFrame:
    d = _matrix(frame.data)
    out = np.zeros_like(d)
    raise_for(fn(_ptr(d), C.c_uint64(d.shape[0]), C.c_uint64(d.shape[1]), *extra, _ptr(out)))
    return RadarFrame(out, frame.fast_rate, frame.prf)


def remove_dc(frame: RadarFrame) -> RadarFrame:
    return _frame_op(N.lib.uwb_remove_dc, frame)


def detrend_linear(frame: RadarFrame) -> RadarFrame:
    return _frame_op(N.lib.uwb_detrend_linear, frame)


def mean_filter_slow(frame: RadarFrame, window: int) -> RadarFrame:
    return _frame_op(N.lib.uwb_mean_filter_slow, frame, C.c_uint64(window))


def subtract_slow_time_mean(frame: RadarFrame) -> RadarFrame:
    return _frame_op(N.lib.uwb_subtract_slow_time_mean, frame)


def normalize_slow(frame: RadarFrame, epsilon: float) -> RadarFrame:
    return _frame_op(N.lib.uwb_normalize_slow, frame, C.c_double(epsilon))


def slow_time_spectrum(frame: RadarFrame, fft_length: int) -> RangeFrequencyMap:
    d = _matrix(frame.data)
    m, n = d.shape
    bins = fft_length // 2 + 1
    power = np.zeros((m, bins))
    freq = np.zeros(bins)
    rng = np.zeros(m)
    raise_for(N.lib.uwb_slow_time_spectrum(_ptr(d), C.c_uint64(m), C.c_uint64(n),
                                           C.c_double(frame.fast_rate), C.c_double(frame.prf),
                                           C.c_uint64(fft_length), _ptr(power), _ptr(freq), _ptr(rng)))
    return RangeFrequencyMap(power, freq, rng)


def band_select(spectrum: RangeFrequencyMap, band_low_hz: float, band_high_hz: float) -> RangeFrequencyMap:
    p = _matrix(spectrum.power)
    f = np.ascontiguousarray(spectrum.freq_axis, dtype=np.float64)
    m, bins = p.shape
    first, kept = C.c_uint64(), C.c_uint64()
    raise_for(N.lib.uwb_band_select(_ptr(p), C.c_uint64(m), C.c_uint64(bins), _ptr(f),
                                    C.c_double(band_low_hz), C.c_double(band_high_hz),
                                    C.byref(first), C.byref(kept), None, None))
    k = kept.value
    out = np.zeros((m, k))
    of = np.zeros(k)
    raise_for(N.lib.uwb_band_select(_ptr(p), C.c_uint64(m), C.c_uint64(bins), _ptr(f),
                                    C.c_double(band_low_hz), C.c_double(band_high_hz),
                                    C.byref(first), C.byref(kept), _ptr(out), _ptr(of)))
    return RangeFrequencyMap(out, of, np.asarray(spectrum.range_axis, dtype=np.float64).copy())


def detect(frame: RadarFrame, config: PipelineConfig, threads: int = 1) -> DetectOutput:
    """pipeline.hpp:79-80; stage errors carry the stage name."""
    d = _matrix(frame.data)
    m, n = d.shape
    L = config.effective_fft_length(n)
    cap = L // 2 + 1
    band = np.zeros(m * cap)
    freq = np.zeros(cap)
    rng = np.zeros(m)
    mask = np.zeros(m * cap, np.uint8)
    thr = np.zeros(m * cap)
    dets = np.zeros(max(1, m * cap), DETECTION_DTYPE)
    kept, nd = C.c_uint64(), C.c_uint64()
    cfg = config.to_c()
    raise_for(N.lib.uwb_detect(_ptr(d), C.c_uint64(m), C.c_uint64(n), C.c_double(frame.fast_rate),
                               C.c_double(frame.prf), C.byref(cfg), C.c_uint64(cap), _ptr(band),
                               _ptr(freq), _ptr(rng), C.byref(kept), _ptr(mask), _ptr(thr), _ptr(dets),
                               C.c_uint64(dets.size), C.byref(nd)))
    k = kept.value
    bm = RangeFrequencyMap(band[: m * k].reshape(m, k).copy(), freq[:k].copy(), rng)
    res = DetectionResult(mask[: m * k].reshape(m, k).copy(), thr[: m * k].reshape(m, k).copy(),
                          dets[: nd.value].copy())
    return DetectOutput(bm, res)


__all__ = [
    "CfarParams", "CellRect", "TrainingWindow", "DetectionResult", "alpha_factor", "training_window",
    "cfar2d_naive", "cfar2d_integral", "SummedAreaTable", "build_sat", "RadarFrame", "PipelineConfig",
    "RangeFrequencyMap", "DetectOutput", "remove_dc", "detrend_linear", "mean_filter_slow",
    "subtract_slow_time_mean", "normalize_slow", "slow_time_spectrum", "band_select", "detect",
    "DETECTION_DTYPE", "CapacityError",
]
