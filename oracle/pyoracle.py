"""TEST INFRASTRUCTURE ONLY: ctypes bindings to the two CPU checkers.

* :class:`RefLib` loads ``oracle/_ref/libuwbref.so``: the reference C++ sources
  (/root/reference/proj/src/{sat,cfar,pipeline,synth}.cpp) compiled unchanged by
  ``oracle/Makefile`` plus the extern "C" shim ``oracle/ref_capi.cpp``.
* :class:`OracleLib` loads ``oracle/_build/libuwboracle.so``: the plain-C
  restatement ``oracle/uwb_oracle.c`` (per-axis windows, slab-local tables).

Errors surface as :class:`OracleError` carrying the reference exception class
name in ``kind`` (errors.hpp:9-47).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libuwbref.so")
ORACLE_SO = os.path.join(HERE, "_build", "libuwboracle.so")

KINDS = {
    1: "DimensionError",
    2: "InputError",
    3: "ParameterError",
    4: "BoundsError",
    5: "ConfigurationError",
    7: "FormatError",
    9: "Error",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, message: str = ""):
        super().__init__(f"{KINDS.get(code, 'Error')}: {message}")
        self.code = code
        self.kind = KINDS.get(code, "Error")
        self.message = message


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


DET_DTYPE = np.dtype([("row", np.uint64), ("col", np.uint64), ("value", np.float64),
                      ("threshold", np.float64)])


@dataclass
class CfarResult:
    mask: np.ndarray            # uint8 rows x cols
    threshold_map: np.ndarray   # float64 rows x cols
    detections: np.ndarray      # DET_DTYPE, sorted value desc, row, col asc


class _PipelineConfig(C.Structure):
    _fields_ = [("mean_filter_window", C.c_uint64), ("fft_length", C.c_uint64),
                ("band_low_hz", C.c_double), ("band_high_hz", C.c_double),
                ("guard_radius", C.c_int), ("background_radius", C.c_int),
                ("pfa", C.c_double), ("backend", C.c_int),
                ("normalization_epsilon", C.c_double), ("mean_filter_mode", C.c_int)]


class _SceneConfig(C.Structure):
    _fields_ = [("m_samples", C.c_uint64), ("n_traces", C.c_uint64),
                ("fast_rate", C.c_double), ("prf", C.c_double),
                ("target_range_m", C.c_double), ("resp_freq_hz", C.c_double),
                ("resp_displacement_m", C.c_double), ("wall_range_m", C.c_double),
                ("wall_amplitude", C.c_double), ("noise_sigma", C.c_double),
                ("pulse_center_hz", C.c_double), ("pulse_bandwidth_hz", C.c_double),
                ("target_attenuation", C.c_double), ("seed", C.c_uint64)]


class RefLib:
    """The reference implementation itself (compiled from /root/reference)."""

    _lib = None

    def __init__(self, path: str = REF_SO):
        if RefLib._lib is None:
            if not os.path.exists(path):
                raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` "
                                        "where /root/reference is mounted")
            RefLib._lib = C.CDLL(path)
        self.lib = RefLib._lib
        self.err = C.create_string_buffer(1024)

    def _check(self, code: int):
        if code != 0:
            raise OracleError(code, self.err.value.decode())

    def build_sat(self, src) -> np.ndarray:
        src = _f64(src)
        rows, cols = src.shape
        out = np.zeros((rows + 1, cols + 1), dtype=np.float64)
        self._check(self.lib.uwbref_build_sat(_p(src), C.c_uint64(rows), C.c_uint64(cols),
                                              _p(out), self.err, C.c_uint64(1024)))
        return out

    def region_sum(self, src, r0, r1, c0, c1) -> float:
        src = _f64(src)
        out = C.c_double()
        self._check(self.lib.uwbref_region_sum(
            _p(src), C.c_uint64(src.shape[0]), C.c_uint64(src.shape[1]), C.c_uint64(r0),
            C.c_uint64(r1), C.c_uint64(c0), C.c_uint64(c1), C.byref(out), self.err,
            C.c_uint64(1024)))
        return out.value

    def alpha_factor(self, n: int, pfa: float) -> float:
        out = C.c_double()
        self._check(self.lib.uwbref_alpha_factor(C.c_uint64(n), C.c_double(pfa), C.byref(out),
                                                 self.err, C.c_uint64(1024)))
        return out.value

    def interior_train_count(self, g: int, b: int) -> int:
        out = C.c_uint64()
        self.lib.uwbref_interior_train_count(C.c_int(g), C.c_int(b), C.byref(out))
        return out.value

    def training_window(self, g, b, pfa, row, col, rows, cols):
        out = np.zeros(9, dtype=np.uint64)
        self._check(self.lib.uwbref_training_window(
            C.c_int(g), C.c_int(b), C.c_double(pfa), C.c_uint64(row), C.c_uint64(col),
            C.c_uint64(rows), C.c_uint64(cols), _p(out), self.err, C.c_uint64(1024)))
        o = [int(v) for v in out]
        return {"outer": tuple(o[0:4]), "guard": tuple(o[4:8]), "n_train": o[8]}

    def cfar2d(self, power_map, g: int, b: int, pfa: float, backend: str = "integral",
               threads: int = 1, det_cap: int | None = None, thresholds: bool = True) -> CfarResult:
        """cfar2d_naive / cfar2d_integral (cfar.cpp:200-227). ``det_cap`` bounds
        the exported list (default: every cell); ``thresholds=False`` skips the
        threshold-map export (``threshold_map`` is then None)."""
        m = _f64(power_map)
        if m.ndim != 2:
            raise ValueError("2-D map required")
        rows, cols = m.shape
        cells = rows * cols
        mask = np.zeros((rows, cols), dtype=np.uint8)
        thr = np.zeros((rows, cols), dtype=np.float64) if thresholds else None
        n_det = C.c_uint64()
        cap = cells if det_cap is None else int(det_cap)
        dr = np.zeros(max(cap, 1), np.uint64)
        dc = np.zeros(max(cap, 1), np.uint64)
        dv = np.zeros(max(cap, 1), np.float64)
        dt = np.zeros(max(cap, 1), np.float64)
        self._check(self.lib.uwbref_cfar2d(
            C.c_int(0 if backend == "naive" else 1), _p(m), C.c_uint64(rows), C.c_uint64(cols),
            C.c_int(g), C.c_int(b), C.c_double(pfa), C.c_uint(threads), _p(mask),
            _p(thr) if thr is not None else None,
            C.byref(n_det), C.c_uint64(cap), _p(dr), _p(dc), _p(dv), _p(dt), self.err,
            C.c_uint64(1024)))
        n = n_det.value
        if n > cap:
            raise OracleError(9, f"{n} detections > det_cap {cap}")
        dets = np.zeros(n, dtype=DET_DTYPE)
        dets["row"], dets["col"], dets["value"], dets["threshold"] = dr[:n], dc[:n], dv[:n], dt[:n]
        return CfarResult(mask, thr, dets)

    def time_cfar_batch(self, maps_f32: np.ndarray, g, b, pfa, workers: int,
                        ref_threads: int = 1):
        maps = np.ascontiguousarray(maps_f32, dtype=np.float32)
        n_maps, rows, cols = maps.shape
        counts = np.zeros(n_maps, dtype=np.uint64)
        secs = C.c_double()
        self._check(self.lib.uwbref_time_cfar_batch(
            _p(maps), C.c_uint64(n_maps), C.c_uint64(rows), C.c_uint64(cols), C.c_int(g),
            C.c_int(b), C.c_double(pfa), C.c_uint(workers), C.c_uint(ref_threads), _p(counts),
            C.byref(secs), self.err, C.c_uint64(1024)))
        return secs.value, counts

    _OPS = {"remove_dc": 0, "detrend_linear": 1, "mean_filter_slow": 2,
            "subtract_slow_time_mean": 3, "normalize_slow": 4}

    def frame_stage(self, op: str, data, window: int = 1, epsilon: float = 1e-12):
        d = _f64(data)
        out = np.zeros_like(d)
        self._check(self.lib.uwbref_frame_stage(
            C.c_int(self._OPS[op]), _p(d), C.c_uint64(d.shape[0]), C.c_uint64(d.shape[1]),
            C.c_uint64(window), C.c_double(epsilon), _p(out), self.err, C.c_uint64(1024)))
        return out

    def slow_time_spectrum(self, data, fft_length: int, prf: float = 68.6,
                           fast_rate: float = 39e9):
        d = _f64(data)
        m = d.shape[0]
        bins = fft_length // 2 + 1
        power = np.zeros((m, bins))
        freq = np.zeros(bins)
        rng = np.zeros(m)
        self._check(self.lib.uwbref_slow_time_spectrum(
            _p(d), C.c_uint64(m), C.c_uint64(d.shape[1]), C.c_double(fast_rate),
            C.c_double(prf), C.c_uint64(fft_length), _p(power), _p(freq), _p(rng), self.err,
            C.c_uint64(1024)))
        return power, freq, rng

    def band_select(self, power, freq_axis, low, high):
        p = _f64(power)
        f = _f64(freq_axis)
        m, bins = p.shape
        out = np.zeros((m, bins))
        of = np.zeros(bins)
        kept = C.c_uint64()
        self._check(self.lib.uwbref_band_select(
            _p(p), C.c_uint64(m), C.c_uint64(bins), _p(f), C.c_double(low), C.c_double(high),
            _p(out), _p(of), C.byref(kept), self.err, C.c_uint64(1024)))
        k = kept.value
        return np.ascontiguousarray(out.reshape(-1)[: m * k].reshape(m, k)), of[:k].copy()

    def detect(self, data, fast_rate=39e9, prf=68.6, mean_filter_window=5, fft_length=0,
               band_low_hz=0.3, band_high_hz=0.8, guard_radius=4, background_radius=8,
               pfa=1e-3, backend="integral", normalization_epsilon=1e-12,
               mean_filter_mode="smoothing", threads=1):
        d = _f64(data)
        m, n = d.shape
        cfg = _PipelineConfig(mean_filter_window, fft_length, band_low_hz, band_high_hz,
                              guard_radius, background_radius, pfa,
                              0 if backend == "naive" else 1, normalization_epsilon,
                              0 if mean_filter_mode == "smoothing" else 1)
        L = fft_length if fft_length else 1 << max(0, (n - 1).bit_length())
        cap = L // 2 + 1
        band = np.zeros(m * cap)
        freq = np.zeros(cap)
        rng = np.zeros(m)
        kcols = C.c_uint64()
        mask = np.zeros(m * cap, np.uint8)
        thr = np.zeros(m * cap)
        n_det = C.c_uint64()
        dcap = m * cap
        dr = np.zeros(dcap, np.uint64)
        dc = np.zeros(dcap, np.uint64)
        dv = np.zeros(dcap)
        dt = np.zeros(dcap)
        self._check(self.lib.uwbref_detect(
            _p(d), C.c_uint64(m), C.c_uint64(n), C.c_double(fast_rate), C.c_double(prf),
            C.byref(cfg), C.c_uint(threads), C.c_uint64(cap), _p(band), _p(freq), _p(rng),
            C.byref(kcols), _p(mask), _p(thr), C.byref(n_det), C.c_uint64(dcap), _p(dr), _p(dc),
            _p(dv), _p(dt), self.err, C.c_uint64(1024)))
        k = kcols.value
        nd = n_det.value
        dets = np.zeros(nd, dtype=DET_DTYPE)
        dets["row"], dets["col"], dets["value"], dets["threshold"] = dr[:nd], dc[:nd], dv[:nd], dt[:nd]
        return {
            "band_power": band[: m * k].reshape(m, k).copy(),
            "freq_axis": freq[:k].copy(),
            "range_axis": rng.copy(),
            "result": CfarResult(mask[: m * k].reshape(m, k).copy(),
                                 thr[: m * k].reshape(m, k).copy(), dets),
        }

    def default_scene_config(self) -> dict:
        c = _SceneConfig()
        self.lib.uwbref_default_scene_config(C.byref(c))
        return {name: getattr(c, name) for name, _ in _SceneConfig._fields_}

    def read_frame(self, path: str):
        """frame_io.cpp:69-122 read_frame_file -> (data m x n, fast_rate, prf)."""
        m, n = C.c_uint32(), C.c_uint32()
        fr, pr = C.c_double(), C.c_double()
        # first call sizes the frame, second copies it
        self._check(self.lib.uwbref_read_frame(path.encode(), None, C.c_uint64(0), C.byref(m), C.byref(n),
                                               C.byref(fr), C.byref(pr), self.err, C.c_uint64(1024)))
        data = np.zeros((m.value, n.value))
        self._check(self.lib.uwbref_read_frame(path.encode(), _p(data), C.c_uint64(data.size), C.byref(m),
                                               C.byref(n), C.byref(fr), C.byref(pr), self.err, C.c_uint64(1024)))
        return data, fr.value, pr.value

    def generate_scene(self, **overrides):
        cfg = self.default_scene_config()
        cfg.update(overrides)
        c = _SceneConfig(**cfg)
        data = np.zeros((int(cfg["m_samples"]), int(cfg["n_traces"])))
        tb = C.c_uint64()
        tf = C.c_double()
        self._check(self.lib.uwbref_generate_scene(C.byref(c), _p(data), C.byref(tb),
                                                   C.byref(tf), self.err, C.c_uint64(1024)))
        return data, {"target_range_bin": tb.value, "resp_freq_hz": tf.value,
                      "prf": cfg["prf"], "fast_rate": cfg["fast_rate"]}


class _Params(C.Structure):
    _fields_ = [("guard_rows", C.c_int), ("guard_cols", C.c_int),
                ("background_rows", C.c_int), ("background_cols", C.c_int),
                ("pfa", C.c_double)]


class _Det(C.Structure):
    _fields_ = [("row", C.c_uint64), ("col", C.c_uint64), ("value", C.c_double),
                ("threshold", C.c_double)]


class OracleLib:
    """The plain-C restatement (oracle/uwb_oracle.c)."""

    _lib = None

    def __init__(self, path: str = ORACLE_SO):
        if OracleLib._lib is None:
            if not os.path.exists(path):
                raise FileNotFoundError(f"{path} missing: run `make -C oracle restatement`")
            lib = C.CDLL(path)
            lib.uwbo_alpha.restype = C.c_double
            lib.uwbo_interior_train_count.restype = C.c_size_t
            OracleLib._lib = lib
        self.lib = OracleLib._lib

    def build_sat(self, src) -> np.ndarray:
        s = _f64(src)
        rows, cols = s.shape if s.ndim == 2 else (0, 0)
        out = np.zeros((rows + 1, cols + 1))
        br, bc = C.c_int64(-1), C.c_int64(-1)
        code = self.lib.uwbo_build_sat(_p(s), C.c_size_t(rows), C.c_size_t(cols), _p(out),
                                       C.byref(br), C.byref(bc))
        if code:
            raise OracleError(code, f"cell ({br.value}, {bc.value})")
        return out

    def alpha(self, n: int, pfa: float) -> float:
        return self.lib.uwbo_alpha(C.c_size_t(n), C.c_double(pfa))

    def interior_train_count(self, gr, gc, br, bc) -> int:
        p = _Params(gr, gc, br, bc, 0.5)
        return int(self.lib.uwbo_interior_train_count(C.byref(p)))

    def cfar(self, power_map, guard_rows, guard_cols, background_rows, background_cols, pfa,
             backend="integral", row_begin=0, row_end=None, slab_local=False,
             det_cap: int | None = None) -> CfarResult:
        m = _f64(power_map)
        rows, cols = m.shape
        row_end = rows if row_end is None else row_end
        p = _Params(guard_rows, guard_cols, background_rows, background_cols, pfa)
        mask = np.zeros((rows, cols), np.uint8)
        thr = np.zeros((rows, cols))
        cap = max(rows * cols, 1) if det_cap is None else int(det_cap)
        dets = (_Det * cap)()
        n_det = C.c_size_t()
        br, bc = C.c_int64(-1), C.c_int64(-1)
        code = self.lib.uwbo_cfar(
            _p(m), C.c_size_t(rows), C.c_size_t(cols), C.byref(p),
            C.c_int(0 if backend == "naive" else 1), C.c_size_t(row_begin), C.c_size_t(row_end),
            C.c_int(1 if slab_local else 0), _p(mask), _p(thr), dets, C.c_size_t(cap),
            C.byref(n_det), C.byref(br), C.byref(bc))
        if code:
            raise OracleError(code, f"cell ({br.value}, {bc.value})")
        n = n_det.value
        if n > cap:
            raise OracleError(9, f"{n} detections > det_cap {cap}")
        arr = np.frombuffer(dets, dtype=DET_DTYPE, count=n).copy()
        return CfarResult(mask, thr, arr)

    def frame_stage(self, op: str, data, window: int = 1, epsilon: float = 1e-12):
        d = _f64(data)
        m, n = d.shape
        out = np.zeros_like(d)
        if op == "remove_dc":
            code = self.lib.uwbo_remove_dc(_p(d), C.c_size_t(m), C.c_size_t(n), _p(out))
        elif op == "detrend_linear":
            code = self.lib.uwbo_detrend_linear(_p(d), C.c_size_t(m), C.c_size_t(n), _p(out))
        elif op == "mean_filter_slow":
            code = self.lib.uwbo_mean_filter_slow(_p(d), C.c_size_t(m), C.c_size_t(n),
                                                  C.c_size_t(window), _p(out))
        elif op == "subtract_slow_time_mean":
            code = self.lib.uwbo_subtract_slow_time_mean(_p(d), C.c_size_t(m), C.c_size_t(n),
                                                         _p(out))
        elif op == "normalize_slow":
            code = self.lib.uwbo_normalize_slow(_p(d), C.c_size_t(m), C.c_size_t(n),
                                                C.c_double(epsilon), _p(out))
        else:
            raise ValueError(op)
        if code:
            raise OracleError(code, op)
        return out

    def slow_time_spectrum(self, data, fft_length: int) -> np.ndarray:
        d = _f64(data)
        m, n = d.shape
        power = np.zeros((m, fft_length // 2 + 1))
        code = self.lib.uwbo_slow_time_spectrum(_p(d), C.c_size_t(m), C.c_size_t(n),
                                                C.c_size_t(fft_length), _p(power))
        if code:
            raise OracleError(code, "slow_time_spectrum")
        return power

    def band_range(self, fft_length, prf, low, high):
        first, kept = C.c_size_t(), C.c_size_t()
        code = self.lib.uwbo_band_range(C.c_size_t(fft_length), C.c_double(prf), C.c_double(low),
                                        C.c_double(high), C.byref(first), C.byref(kept))
        if code:
            raise OracleError(code, "band_select")
        return first.value, kept.value

    def detect(self, data, prf=68.6, mean_filter_window=5, fft_length=0, band_low_hz=0.3,
               band_high_hz=0.8, guard_rows=4, guard_cols=None, background_rows=8,
               background_cols=None, pfa=1e-3, normalization_epsilon=1e-12,
               mean_filter_mode="smoothing"):
        """pipeline.cpp:246-275 restated (integral backend)."""
        d = _f64(data)
        m, n = d.shape
        L = fft_length if fft_length else 1 << max(0, (n - 1).bit_length())
        x = self.frame_stage("remove_dc", d)
        x = self.frame_stage("detrend_linear", x)
        if mean_filter_mode == "smoothing":
            x = self.frame_stage("mean_filter_slow", x, window=mean_filter_window)
        else:
            x = self.frame_stage("subtract_slow_time_mean", x)
        x = self.frame_stage("normalize_slow", x, epsilon=normalization_epsilon)
        power = self.slow_time_spectrum(x, L)
        first, kept = self.band_range(L, prf, band_low_hz, band_high_hz)
        band = np.ascontiguousarray(power[:, first:first + kept])
        gc = guard_rows if guard_cols is None else guard_cols
        bc = background_rows if background_cols is None else background_cols
        res = self.cfar(band, guard_rows, gc, background_rows, bc, pfa)
        freq = np.arange(first, first + kept, dtype=np.float64) * prf / L
        return {"band_power": band, "freq_axis": freq, "first_bin": first, "result": res}
