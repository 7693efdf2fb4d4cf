"""RFRM ingest: the parser's checks and messages against the
reference's read_frame (oracle/_ref, frame_io.cpp compiled unchanged), on CPU;
the device transpose and the file -> batched detect chain on the GPU."""
import struct

import numpy as np
import pytest

from oracle.pyoracle import OracleError


def _image(m=4, n=3, version=1, fast_rate=39e9, prf=20.0, payload=None, extra=b""):
    head = b"RFRM" + struct.pack("<HIIdd", version, m, n, fast_rate, prf)
    if payload is None:
        payload = np.arange(m * n, dtype="<f4").tobytes()
    return head + payload + extra


BAD = {
    "bad magic": b"RFRX" + _image()[4:],
    "short magic": b"RF",
    "truncated header": _image()[:12],
    "unsupported version": _image(version=2),
    "too small": _image(m=1, n=5, payload=np.zeros(5, "<f4").tobytes()),
    "truncated payload": _image()[:-3],
    "trailing bytes": _image(extra=b"\x00"),
    "bad prf": _image(prf=0.0),
    "nan rate": _image(fast_rate=float("nan")),
}


@pytest.mark.parametrize("case", sorted(BAD))
def test_parse_errors_match_reference(uwb, ref, tmp_path, case):
    from paper_2012_11077_b200 import ingest
    path = tmp_path / "f.rfrm"
    path.write_bytes(BAD[case])
    with pytest.raises(OracleError) as r:
        ref.read_frame(str(path))
    assert r.value.kind == "FormatError"
    with pytest.raises(uwb.FormatError) as g:
        ingest.parse(BAD[case])
    assert str(g.value) == r.value.message


def test_parse_good_file_and_writer_round_trip(uwb, ref, tmp_path):
    from paper_2012_11077_b200 import ingest
    rng = np.random.default_rng(3)
    data = rng.standard_normal((6, 5)).astype(np.float32).astype(np.float64)
    path = tmp_path / "ok.rfrm"
    ingest.write_frame(path, data, 39e9, 68.6)
    info = ingest.parse(path.read_bytes())
    assert (info.m_samples, info.n_traces, info.fast_rate, info.prf) == (6, 5, 39e9, 68.6)
    assert info.payload_offset == 30 and info.payload_bytes == 120
    got, fr, pr = ref.read_frame(str(path))
    assert np.array_equal(got, data) and (fr, pr) == (39e9, 68.6)


@pytest.mark.gpu
def test_device_transpose_and_detect_from_files(uwb, ref, cuda, tmp_path):
    import torch
    from paper_2012_11077_b200 import ingest, synth
    from paper_2012_11077_b200.batch import DetectBatch
    paths = []
    for i in range(3):
        rec = synth.cfg2_record(seed=90 + i, device="cpu").double().numpy()
        p = tmp_path / f"r{i}.rfrm"
        ingest.write_frame(p, rec, 39e9, 20.0)
        paths.append(str(p))
    fb = ingest.read_frames(paths, device=cuda, dtype=torch.float32)
    assert fb.frames.shape == (3, 512, 1024) and fb.prf == 20.0
    config = uwb.PipelineConfig(mean_filter_window=5, fft_length=1024, cfar=uwb.CfarParams(1, 4, 1e-3))
    db = DetectBatch(3, 512, 1024, config, prf=fb.prf, fast_rate=fb.fast_rate, dtype=torch.float32)
    db(fb.frames)
    torch.cuda.synchronize()
    for i, p in enumerate(paths):
        data, fr, pr = ref.read_frame(p)
        assert np.array_equal(fb.frames[i].double().cpu().numpy(), data)
        exp = ref.detect(data, fast_rate=fr, prf=pr, mean_filter_window=5, fft_length=1024, guard_radius=1,
                         background_radius=4, pfa=1e-3)
        assert np.array_equal(db.mask(i), exp["result"].mask)
        assert np.array_equal(db.band[i].cpu().numpy(), exp["band_power"])
    # odd shapes and fp64 output
    rng = np.random.default_rng(4)
    odd = rng.standard_normal((37, 70))
    p = tmp_path / "odd.rfrm"
    ingest.write_frame(p, odd, 1e9, 10.0)
    f64 = ingest.read_frames([str(p)], device=cuda, dtype=torch.float64)
    data, _, _ = ref.read_frame(str(p))
    assert np.array_equal(f64.frames[0].cpu().numpy(), data)
    bad = odd.copy()
    bad[3, 4] = np.inf
    ingest.write_frame(p, bad, 1e9, 10.0)
    with pytest.raises(uwb.FormatError, match="non-finite sample"):
        ingest.read_frames([str(p)], device=cuda)
