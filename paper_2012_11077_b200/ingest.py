"""RFRM frame files onto the device (frame_io.hpp:10-23).

``read_frames`` validates every file image exactly as the reference's
read_frame does (frame_io.cpp:69-122, same FormatError messages, via
uwb_rfrm_parse), packs the trace-major f32 payloads back to back in pinned host
memory, copies them to the device as they lie and transposes them there into
range-major frames (uwb_dev_rfrm_to_frames), ready for DetectBatch. Values are
the file's f32 samples widened exactly, so the frames equal the reference's
in-memory RadarFrame::data bit for bit.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import FormatError, raise_for


@dataclass
class FrameBatch:
    frames: torch.Tensor     # (n_records, m_samples, n_traces) on the device
    fast_rate: float
    prf: float


def parse(image: bytes | np.ndarray) -> N.uwb_rfrm_info:
    """Validate one RFRM file image; raises FormatError with the reference's text."""
    buf = np.frombuffer(image, dtype=np.uint8) if not isinstance(image, np.ndarray) else image
    info = N.uwb_rfrm_info()
    raise_for(N.lib.uwb_rfrm_parse(buf.ctypes.data_as(C.c_void_p), buf.size, C.byref(info)))
    return info


def read_frames(paths, device=None, dtype: torch.dtype = torch.float32) -> FrameBatch:
    """Read RFRM files of one shape into a device batch (n, m_samples, n_traces)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    images = []
    for p in paths:
        try:
            images.append(np.fromfile(p, dtype=np.uint8))
        except OSError:
            raise FormatError(f"frame file: cannot open '{p}'") from None
    infos = [parse(im) for im in images]
    if not infos:
        raise ValueError("no frame files")
    m, n = infos[0].m_samples, infos[0].n_traces
    if any((i.m_samples, i.n_traces) != (m, n) for i in infos):
        raise ValueError("all frames of a batch must have the same shape")
    pinned = torch.empty(len(images) * m * n, dtype=torch.float32, pin_memory=True)
    host = pinned.numpy().view(np.uint8)
    per = m * n * 4
    for k, (im, inf) in enumerate(zip(images, infos)):
        host[k * per:(k + 1) * per] = im[inf.payload_offset:inf.payload_offset + per]
    payload = pinned.to(dev, non_blocking=True)
    frames = torch.empty((len(images), m, n), dtype=dtype, device=dev)
    bad = torch.empty(len(images), dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream(dev)
    raise_for(N.lib.uwb_dev_rfrm_to_frames(payload.data_ptr(), len(images), m, n,
                                           N.UWB_F32 if dtype == torch.float32 else N.UWB_F64, frames.data_ptr(),
                                           bad.data_ptr(), C.c_void_p(s.cuda_stream)))
    if (bad.cpu().numpy().astype(np.uint64) != np.uint64(0xFFFFFFFFFFFFFFFF)).any():
        raise FormatError("frame file: RadarFrame: non-finite sample")
    return FrameBatch(frames, float(infos[0].fast_rate), float(infos[0].prf))


def write_frame(path, data: np.ndarray, fast_rate: float, prf: float, version: int = 1) -> None:
    """frame_io.cpp:45-59 (for tests and tools): header + trace-major f32 payload."""
    d = np.asarray(data, dtype=np.float64)
    m, n = d.shape
    with open(path, "wb") as f:
        f.write(b"RFRM" + struct.pack("<HIIdd", version, m, n, fast_rate, prf))
        f.write(np.ascontiguousarray(d.T, dtype="<f4").tobytes())
