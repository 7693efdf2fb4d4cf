"""Device-resident batched CA-CFAR (the throughput path) over torch CUDA tensors.

One :class:`BatchCfar` owns every device buffer of a batch shape (alpha table,
bit-packed masks, detection lists, counts, workspace) so repeated calls launch
kernels only: SAT (kernel c) -> CFAR (kernel d) -> per-map detection sort, on
the caller's current torch stream. PyTorch is used for allocation and streams
only; all arithmetic is in libuwbvital_b200.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .api import DETECTION_DTYPE, CfarParams
from .errors import CapacityError, InputError, raise_for

_DT = {torch.float32: N.UWB_F32, torch.float64: N.UWB_F64}
_MODES = {"global": N.UWB_SAT_GLOBAL, "slab": N.UWB_SAT_SLAB, "tile": N.UWB_SAT_TILE}


class BatchCfar:
    def __init__(self, n_maps: int, rows: int, cols: int, params: CfarParams,
                 dtype: torch.dtype = torch.float32, sat_mode: str = "global", slab_rows: int = 0,
                 det_capacity: int = 1024, device=None, want_mask_u8: bool = False,
                 want_thresholds: bool = False, window: tuple[int, int, int, int] | None = None,
                 workspace: torch.Tensor | None = None, tie_capacity: int = 64):
        """``window = (global_rows, buf_row0, row_begin, row_end[, col_bands])``: the
        maps passed to each call hold rows [buf_row0, buf_row0 + rows) of maps with
        ``global_rows`` rows and the call owns rows [row_begin, row_end) (one
        rank's row slab); outputs then cover the owned rows only.
        ``col_bands`` > 0 also gives every band of that many columns its own
        table (``sat_mode="tile"`` semantics)."""
        if dtype not in _DT:
            raise ValueError("maps must be float32 or float64")
        params.validate()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.n_maps, self.rows, self.cols = int(n_maps), int(rows), int(cols)
        self.params = params
        self.dtype = dtype
        self.sat_mode = _MODES[sat_mode]
        self.slab_rows = int(slab_rows)
        self.det_capacity = int(det_capacity)
        self.words_per_row = (self.cols + 31) // 32
        self.window = None if window is None else N.uwb_row_window(*(int(x) for x in tuple(window) + (0,) * (5 - len(window))))
        out_rows = self.rows if window is None else int(window[3]) - int(window[2])
        self.out_rows = out_rows
        dev = self.device
        self.alpha = torch.from_numpy(params.alpha_table()).to(dev)
        self.mask_bits = torch.zeros((self.n_maps, out_rows, self.words_per_row), dtype=torch.int32, device=dev)
        self.dets = torch.zeros((self.n_maps, max(1, self.det_capacity), 32), dtype=torch.uint8, device=dev)
        self.counts = torch.zeros(self.n_maps, dtype=torch.int64, device=dev)
        self.first_bad = torch.zeros((self.n_maps, 2), dtype=torch.int64, device=dev)
        self.mask_u8 = (torch.zeros((self.n_maps, out_rows, self.cols), dtype=torch.uint8, device=dev)
                        if want_mask_u8 else None)
        self.thresholds = (torch.zeros((self.n_maps, out_rows, self.cols), dtype=torch.float64, device=dev)
                           if want_thresholds else None)
        # tie band (|cut - T| <= 1e-6 T) and per-map certificate status (certified path)
        self.tie_capacity = int(tie_capacity)
        self.tie_counts = torch.zeros(self.n_maps, dtype=torch.int64, device=dev)
        self.ties = torch.zeros((self.n_maps, max(1, self.tie_capacity), 32), dtype=torch.uint8, device=dev)
        self.cert_status = torch.zeros(self.n_maps, dtype=torch.int32, device=dev)
        self._cparams = params.to_c()
        self._batch = N.uwb_map_batch(None, _DT[dtype], 0, self.n_maps, self.rows, self.cols, self.cols,
                                      self.rows * self.cols)
        if self.window is None:
            ws = N.lib.uwb_dev_cfar2d_workspace(C.byref(self._batch), C.byref(self._cparams), self.sat_mode,
                                                C.c_uint64(self.slab_rows), C.c_uint64(self.det_capacity))
        else:
            ws = N.lib.uwb_dev_cfar2d_window_workspace(C.byref(self._batch), C.byref(self.window),
                                                       C.byref(self._cparams), C.c_uint64(self.slab_rows),
                                                       C.c_uint64(self.det_capacity))
        if workspace is not None:  # shared with another BatchCfar (table reuse, see __call__)
            if workspace.numel() < int(ws) or workspace.dtype != torch.uint8:
                raise ValueError(f"workspace needs {int(ws)} bytes")
            self.workspace = workspace
        else:
            self.workspace = torch.empty(int(ws), dtype=torch.uint8, device=dev)
        self._out = N.uwb_cfar_outputs(
            self.mask_bits.data_ptr(), self.words_per_row, out_rows * self.words_per_row,
            self.mask_u8.data_ptr() if self.mask_u8 is not None else None,
            self.thresholds.data_ptr() if self.thresholds is not None else None,
            self.dets.data_ptr(), self.det_capacity, self.counts.data_ptr(), self.first_bad.data_ptr(),
            self.tie_counts.data_ptr(), self.ties.data_ptr(), self.tie_capacity, self.cert_status.data_ptr())

    def __call__(self, maps: torch.Tensor, sort: bool = True, stream=None, phase_events: bool = False,
                 reuse_tables: bool = False, naive: bool = False, fused: bool = False,
                 exact: bool = False, dense_tables: bool = False, fixed_ring_rows: bool = False,
                 certify: bool = False, cta_tables: bool = False) -> None:
        """Launch SAT + CFAR (+ sort) for ``maps`` of shape (n_maps, rows, cols).
        ``phase_events`` records per-phase CUDA events (read with :func:`phase_ms`).
        ``reuse_tables`` skips the SAT: the (shared) workspace already holds the
        tables of these maps from the previous call (another parameter set).
        ``naive`` runs the naive backend (explicit window sums, no table).
        ``fused`` runs SAT and CFAR as one kernel with the table kept on chip
        (whole-map batches; no table is left for ``reuse_tables``).
        ``exact`` forces the two-kernel path (full table, then the ring CFAR)
        instead of the default certified-decision path; a call whose tables a
        later ``reuse_tables`` call reads must pass it. ``dense_tables`` and
        ``fixed_ring_rows`` are test hooks that change the schedule, not the
        results (full tables on the certified path; 256-row ring chunks).
        ``certify`` takes the certified path also for a small batch (which by
        default runs the exact path with one thread-block cluster per table);
        ``cta_tables`` (test hook) builds a small batch's tables with one CTA per
        table instead."""
        if maps.dtype != self.dtype or tuple(maps.shape) != (self.n_maps, self.rows, self.cols):
            raise ValueError(f"expected {(self.n_maps, self.rows, self.cols)} {self.dtype}, got "
                             f"{tuple(maps.shape)} {maps.dtype}")
        if not maps.is_cuda or not maps.is_contiguous():
            raise ValueError("maps must be a contiguous CUDA tensor")
        self._batch.maps = maps.data_ptr()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        flags = (0 if sort else 1) | (2 if phase_events else 0) | (4 if reuse_tables else 0) | (8 if naive else 0) | (16 if fused else 0) | (64 if exact else 0) | (128 if dense_tables else 0) | (256 if fixed_ring_rows else 0) | (512 if certify else 0) | (1024 if cta_tables else 0)
        if self.window is None:
            st = N.lib.uwb_dev_cfar2d(C.byref(self._batch), C.byref(self._cparams), self.alpha.data_ptr(),
                                      self.sat_mode, C.c_uint64(self.slab_rows), C.byref(self._out),
                                      self.workspace.data_ptr(), C.c_uint64(self.workspace.numel()), flags,
                                      C.c_void_p(s.cuda_stream))
        else:
            st = N.lib.uwb_dev_cfar2d_window(C.byref(self._batch), C.byref(self.window), C.byref(self._cparams),
                                             self.alpha.data_ptr(), C.c_uint64(self.slab_rows), C.byref(self._out),
                                             self.workspace.data_ptr(), C.c_uint64(self.workspace.numel()),
                                             flags, C.c_void_p(s.cuda_stream))
        raise_for(st)

    # ---- host views (synchronising) ----
    def check_inputs(self) -> None:
        """Raise the reference's InputError for the first map with a bad cell."""
        fb = self.first_bad.cpu().numpy().astype(np.uint64)
        for i in range(self.n_maps):
            if fb[i, 0] != np.uint64(0xFFFFFFFFFFFFFFFF):
                r, c = divmod(int(fb[i, 0]), self.cols)
                raise InputError(f"build_sat: non-finite entry at ({r}, {c})", r, c)
            if fb[i, 1] != np.uint64(0xFFFFFFFFFFFFFFFF):
                r, c = divmod(int(fb[i, 1]), self.cols)
                raise InputError(f"cfar2d: cell ({r}, {c}) is not a finite non-negative power", r, c)

    def detection_counts(self) -> np.ndarray:
        return self.counts.cpu().numpy()

    def tie_band(self, i: int) -> np.ndarray:
        """Map i's tie-band cells (|cut - T| <= 1e-6 T) from the certified path,
        as detection records {row, col, value=cut, threshold=T}, sorted by (row, col)."""
        n = int(self.tie_counts[i].item())
        if n < 0 or n == 0xFFFFFFFFFFFFFFFF:
            raise RuntimeError(f"map {i}: tie band unknown (the map ran the exact path)")
        if n > self.tie_capacity:
            raise CapacityError(f"map {i}: {n} tie-band cells > capacity {self.tie_capacity}", n)
        raw = self.ties[i, :n].contiguous().cpu().numpy().reshape(-1)
        t = np.frombuffer(raw.tobytes(), dtype=DETECTION_DTYPE, count=n).copy()
        return t[np.lexsort((t["col"], t["row"]))]

    def detections(self, i: int) -> np.ndarray:
        n = int(self.counts[i].item())
        if n > self.det_capacity:
            raise CapacityError(f"map {i}: {n} detections > capacity {self.det_capacity}", n)
        raw = self.dets[i, :n].contiguous().cpu().numpy().reshape(-1)
        return np.frombuffer(raw.tobytes(), dtype=DETECTION_DTYPE, count=n).copy()

    def mask(self, i: int) -> np.ndarray:
        """Unpack map i's bit mask into an (owned rows) x cols uint8 array."""
        words = self.mask_bits[i].cpu().numpy().view(np.uint32)
        bits = np.unpackbits(words.view(np.uint8).reshape(self.out_rows, -1), axis=1, bitorder="little")
        return bits[:, : self.cols].astype(np.uint8)


class DetectBatch:
    """Batched detect() on the device (pipeline.cpp:246-275 per record): the
    front end of every record writes its band power straight into the CFAR's
    input maps, then one CFAR call covers all records. ``records`` passed to a
    call: (n_records, m fast-time rows, n slow-time columns), float32/64, CUDA."""

    def __init__(self, n_records: int, m: int, n: int, config, prf: float, fast_rate: float = 39e9,
                 dtype: torch.dtype = torch.float32, det_capacity: int = 4096, device=None):
        if dtype not in _DT:
            raise ValueError("records must be float32 or float64")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.n_records, self.m, self.n = int(n_records), int(m), int(n)
        self.dtype, self.prf, self.fast_rate = dtype, float(prf), float(fast_rate)
        self.det_capacity = int(det_capacity)
        self._cfg = config.to_c()
        kept = C.c_uint64()
        empty = N.uwb_cfar_outputs()
        raise_for(N.lib.uwb_dev_detect_batch(None, _DT[dtype], 0, self.m, self.n, C.c_double(self.fast_rate),
                                             C.c_double(self.prf), C.byref(self._cfg), None, C.byref(kept),
                                             C.byref(empty), None, 0, 0, None))
        self.kept = int(kept.value)
        dev = self.device
        self.words_per_row = (self.kept + 31) // 32
        self.band = torch.zeros((self.n_records, self.m, self.kept), dtype=torch.float64, device=dev)
        self.mask_bits = torch.zeros((self.n_records, self.m, self.words_per_row), dtype=torch.int32, device=dev)
        self.dets = torch.zeros((self.n_records, max(1, self.det_capacity), 32), dtype=torch.uint8, device=dev)
        self.counts = torch.zeros(self.n_records, dtype=torch.int64, device=dev)
        self.first_bad = torch.zeros((self.n_records, 2), dtype=torch.int64, device=dev)
        ws = N.lib.uwb_dev_detect_batch_workspace(self.n_records, self.m, self.n, C.c_double(self.prf),
                                                  C.byref(self._cfg), self.det_capacity)
        self.workspace = torch.empty(max(int(ws), 16), dtype=torch.uint8, device=dev)
        self._out = N.uwb_cfar_outputs(
            self.mask_bits.data_ptr(), self.words_per_row, self.m * self.words_per_row, None, None,
            self.dets.data_ptr(), self.det_capacity, self.counts.data_ptr(), self.first_bad.data_ptr())

    def __call__(self, records: torch.Tensor, stream=None, general_kernels: bool = False,
                 phase_events: bool = False) -> None:
        """``general_kernels`` (test hook): the per-stage front-end kernels instead
        of the fused two-kernel front end (same results). ``phase_events``
        records the CFAR call's phase events (read with :func:`phase_ms4`)."""
        if records.dtype != self.dtype or tuple(records.shape) != (self.n_records, self.m, self.n):
            raise ValueError(f"expected {(self.n_records, self.m, self.n)} {self.dtype}")
        if not records.is_cuda or not records.is_contiguous():
            raise ValueError("records must be a contiguous CUDA tensor")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        kept = C.c_uint64()
        raise_for(N.lib.uwb_dev_detect_batch(records.data_ptr(), _DT[self.dtype], self.n_records, self.m, self.n,
                                             C.c_double(self.fast_rate), C.c_double(self.prf), C.byref(self._cfg),
                                             self.band.data_ptr(), C.byref(kept), C.byref(self._out),
                                             self.workspace.data_ptr(), C.c_uint64(self.workspace.numel()),
                                             (256 if general_kernels else 0) | (2 if phase_events else 0),
                                             C.c_void_p(s.cuda_stream)))

    def check_inputs(self) -> None:
        """Raise the reference's InputError for the first record with a non-finite sample."""
        fb = self.first_bad.cpu().numpy().astype(np.uint64)
        for i in range(self.n_records):
            if fb[i, 0] != np.uint64(0xFFFFFFFFFFFFFFFF):
                raise InputError("RadarFrame: non-finite sample")

    def detections(self, i: int) -> np.ndarray:
        n = int(self.counts[i].item())
        if n > self.det_capacity:
            raise CapacityError(f"record {i}: {n} detections > capacity {self.det_capacity}", n)
        raw = self.dets[i, :n].contiguous().cpu().numpy().reshape(-1)
        return np.frombuffer(raw.tobytes(), dtype=DETECTION_DTYPE, count=n).copy()

    def mask(self, i: int) -> np.ndarray:
        words = self.mask_bits[i].cpu().numpy().view(np.uint32)
        bits = np.unpackbits(words.view(np.uint8).reshape(self.m, -1), axis=1, bitorder="little")
        return bits[:, : self.kept].astype(np.uint8)


def phase_ms4(max_calls: int = 1024) -> np.ndarray:
    """(calls, 4) array of {certify, sat, cfar, sort} milliseconds (certify is the
    certified path's window-sum pass + tap marking; ~0 on the exact path; cfar is
    the certified resolve or the exact ring kernel)."""
    out = np.zeros((max_calls, 4), dtype=np.float32)
    n = N.lib.uwb_dev_phase_ms4(out.ctypes.data_as(C.c_void_p), max_calls)
    return out[:n].copy()


def phase_ms(max_calls: int = 1024) -> np.ndarray:
    """(calls, 3) array of {sat, cfar, sort} milliseconds of the calls made with
    ``phase_events=True`` since the last read (synchronises on them)."""
    out = np.zeros((max_calls, 3), dtype=np.float32)
    n = N.lib.uwb_dev_phase_ms(out.ctypes.data_as(C.c_void_p), max_calls)
    return out[:n].copy()


def kernel_launches() -> int:
    return int(N.lib.uwb_kernel_launches())


def host_cfar2d_batch(maps_host: torch.Tensor, params: CfarParams, mask_bits_host: torch.Tensor,
                      dets_host: torch.Tensor, counts_host: torch.Tensor, det_capacity: int,
                      sat_mode: str = "global", slab_rows: int = 0, maps_per_chunk: int = 128) -> None:
    """End-to-end call from (pinned) host buffers: H2D, SAT+CFAR+sort, D2H, streamed in chunks."""
    n_maps, rows, cols = maps_host.shape
    b = N.uwb_map_batch(maps_host.data_ptr(), _DT[maps_host.dtype], 0, n_maps, rows, cols, cols, rows * cols)
    p = params.to_c()
    st = N.lib.uwb_host_cfar2d_batch(C.byref(b), C.byref(p), _MODES[sat_mode], C.c_uint64(slab_rows),
                                     mask_bits_host.data_ptr(), dets_host.data_ptr(), C.c_uint64(det_capacity),
                                     counts_host.data_ptr(), C.c_uint64(maps_per_chunk))
    raise_for(st)
