"""GPU parity: front-end stages and detect() vs the reference pipeline.cpp (compiled
in oracle/_ref with the oracle's FFTW provider). Cases follow
proj/tests/test_pipeline.cpp. Stages before the FFT are bit-identical to the
reference; the spectrum is bit-identical to the oracle's FFTW provider and within
the reference tests' 1e-9 of the direct DFT (FFTW itself is absent)."""
import math

import numpy as np
import pytest

from tests.helpers import assert_bitwise, assert_same_result, uniform_frame

pytestmark = pytest.mark.gpu


def F(uwb, data, prf=68.6, fast_rate=39e9):
    return uwb.RadarFrame(np.asarray(data, dtype=np.float64), fast_rate, prf)


@pytest.mark.parametrize("op", ["remove_dc", "detrend_linear", "subtract_slow_time_mean"])
@pytest.mark.parametrize("shape,seed", [((128, 24), 9), ((64, 30), 41), ((200, 2), 3), ((512, 1024), 2)])
def test_stage_bit_identical(uwb, ref, cuda, op, shape, seed):
    d = uniform_frame(*shape, seed)
    got = getattr(uwb, op)(F(uwb, d)).data
    assert_bitwise(got, ref.frame_stage(op, d), op)


@pytest.mark.parametrize("window", [1, 3, 5, 9, 49])
def test_mean_filter_bit_identical(uwb, ref, cuda, window):
    d = uniform_frame(6, 50, 77)
    assert_bitwise(uwb.mean_filter_slow(F(uwb, d), window).data,
                   ref.frame_stage("mean_filter_slow", d, window), f"window {window}")


def test_mean_filter_edges_and_errors(uwb, cuda):  # test_pipeline.cpp:106-138
    d = uniform_frame(4, 25, 1) * 0 + 3.25
    assert (uwb.mean_filter_slow(F(uwb, d), 5).data == 3.25).all()
    d = uniform_frame(4, 20, 5)
    for w in (0, 4, 21):
        with pytest.raises(uwb.ParameterError):
            uwb.mean_filter_slow(F(uwb, d), w)


def test_normalize(uwb, ref, cuda):  # test_pipeline.cpp:150-177
    out = uwb.normalize_slow(F(uwb, [[0.5, -2.0, 1.0]]), 1e-12).data
    assert out.tolist() == [[0.25, -1.0, 0.5]]
    assert (uwb.normalize_slow(F(uwb, np.zeros((3, 10))), 1e-12).data == 0).all()
    d = uniform_frame(12, 33, 1234)
    out = uwb.normalize_slow(F(uwb, d), 1e-12).data
    assert (np.abs(out).max(axis=1) == 1.0).all()
    assert_bitwise(out, ref.frame_stage("normalize_slow", d, 1, 1e-12), "normalize")
    with pytest.raises(uwb.ParameterError):
        uwb.normalize_slow(F(uwb, d), 0.0)


def test_remove_dc_properties(uwb, cuda):  # test_pipeline.cpp:40-69
    assert (uwb.remove_dc(F(uwb, np.full((16, 4), 3.5))).data == 0).all()
    d = np.tile(np.where(np.arange(16) % 2 == 0, 1.0, -1.0)[:, None], (1, 3))
    assert (uwb.remove_dc(F(uwb, d)).data == d).all()


def test_detrend_annihilates_line(uwb, cuda):  # test_pipeline.cpp:71-88
    d = np.tile((2.0 + 0.5 * np.arange(64))[:, None], (1, 3))
    out = uwb.detrend_linear(F(uwb, d)).data
    assert np.abs(out).max() <= 1e-9 * np.abs(d).max()
    assert (uwb.detrend_linear(F(uwb, np.zeros((32, 2)))).data == 0).all()


@pytest.mark.parametrize("n,L", [(64, 64), (50, 64), (600, 1024), (1024, 1024), (100, 128), (600, 600),
                                 (40, 50), (2, 2), (3000, 4096)])
def test_spectrum_matches_reference(uwb, ref, oracle, cuda, n, L):
    d = uniform_frame(3, n, 71)
    got = uwb.slow_time_spectrum(F(uwb, d), L)
    pw, fa, ra = ref.slow_time_spectrum(d, L)
    # bit-identical to the reference compiled with the oracle's FFTW provider
    assert_bitwise(got.power, pw, f"spectrum n={n} L={L}")
    assert_bitwise(got.freq_axis, fa, "freq axis")
    assert_bitwise(got.range_axis, ra, "range axis")
    # and within 1e-9 of the direct DFT (what the reference tests pin against FFTW)
    x = np.zeros((3, L))
    x[:, :n] = d
    exact = np.abs(np.fft.rfft(x, axis=1)) ** 2
    scale = np.maximum(exact, 1e-9 * exact.max(axis=1, keepdims=True))
    assert (np.abs(got.power - exact) / scale).max() < 1e-9


def test_on_bin_cosine(uwb, cuda):  # test_pipeline.cpp:202-220
    n, k0 = 64, 9
    v = np.cos(2 * math.pi * k0 * np.arange(n) / n)
    spec = uwb.slow_time_spectrum(F(uwb, np.vstack([v, v]), prf=64.0), n)
    expect = (n / 2) ** 2
    assert abs(spec.power[0, k0] - expect) <= 1e-9 * expect
    others = np.delete(spec.power[0], k0)
    assert (others <= 1e-9 * expect).all()


def test_spectrum_errors(uwb, cuda):
    with pytest.raises(uwb.ParameterError) as e:
        uwb.slow_time_spectrum(F(uwb, uniform_frame(2, 40, 8)), 39)
    assert str(e.value) == "slow_time_spectrum: fft_length 39 < trace count 40"


def test_band_select_bins(uwb, cuda):  # test_pipeline.cpp:259-292
    d = uniform_frame(4, 600, 15)
    full = uwb.slow_time_spectrum(F(uwb, d, prf=68.6), 1024)
    band = uwb.band_select(full, 0.3, 0.8)
    assert band.freq_axis.size == 7
    assert band.freq_axis[0] == full.freq_axis[5] and band.freq_axis[-1] == full.freq_axis[11]
    assert (band.power == full.power[:, 5:12]).all()
    full = uwb.slow_time_spectrum(F(uwb, uniform_frame(3, 32, 16), prf=32.0), 32)
    band = uwb.band_select(full, 0.0, 16.0)
    assert (band.power == full.power).all()
    full = uwb.slow_time_spectrum(F(uwb, uniform_frame(2, 64, 17), prf=64.0), 64)
    with pytest.raises(uwb.ConfigurationError) as e:
        uwb.band_select(full, 0.1, 0.9)
    assert "resolution" in str(e.value)


def _detect_both(uwb, ref, data, prf=68.6, **cfg):
    g = cfg.pop("guard_radius", 4)
    b = cfg.pop("background_radius", 8)
    pfa = cfg.pop("pfa", 1e-3)
    backend = cfg.pop("backend", "integral")
    config = uwb.PipelineConfig(cfar=uwb.CfarParams(g, b, pfa), backend=backend, **cfg)
    got = uwb.detect(F(uwb, data, prf=prf), config)
    exp = ref.detect(data, prf=prf, guard_radius=g, background_radius=b, pfa=pfa, backend=backend, **cfg)
    return got, exp


@pytest.mark.parametrize("seed", [7, 3, 11])
@pytest.mark.parametrize("backend", ["integral", "naive"])
def test_detect_default_scene_bit_identical(uwb, ref, cuda, seed, backend):  # test_pipeline.cpp:294-342
    data, truth = ref.generate_scene(seed=seed)
    got, exp = _detect_both(uwb, ref, data, backend=backend)
    assert_bitwise(got.band_map.power, exp["band_power"], "band map")
    assert_bitwise(got.band_map.freq_axis, exp["freq_axis"], "freq axis")
    assert_same_result(got.detections, exp["result"], "detect")
    found = any(abs(got.band_map.freq_axis[int(d["col"])] - truth["resp_freq_hz"]) <= 68.6 / 1024 and
                abs(int(d["row"]) - truth["target_range_bin"]) <= 3 for d in got.detections.detections)
    assert found


def test_detect_cfg2_record_bit_identical(uwb, ref, cuda):
    """BASELINE config 2: fp32 raw record 512 x 1024 at 20 Hz, window 5,
    0.3-0.8 Hz band (bins 16..40), CFAR g1 b4 pfa 1e-3."""
    import torch
    from paper_2012_11077_b200 import synth
    rec = synth.cfg2_record(device="cuda").double().cpu().numpy()
    got, exp = _detect_both(uwb, ref, rec, prf=20.0, guard_radius=1, background_radius=4, pfa=1e-3)
    assert got.band_map.power.shape == (512, 25)
    assert_bitwise(got.band_map.power, exp["band_power"], "band map")
    assert_same_result(got.detections, exp["result"], "cfg2 detect")
    rows = got.detections.detections["row"].astype(int)
    assert ((rows >= 190) & (rows <= 210)).any()


def test_detect_modes_and_static_clutter(uwb, ref, cuda):  # test_pipeline.cpp:344-385
    data, _ = ref.generate_scene(noise_sigma=0.0, resp_displacement_m=0.0)
    got, exp = _detect_both(uwb, ref, data, fft_length=data.shape[1])
    assert_bitwise(got.band_map.power, exp["band_power"], "matched-length band map")
    got, exp = _detect_both(uwb, ref, data)
    assert len(got.detections.detections) == 0
    got, exp = _detect_both(uwb, ref, data, mean_filter_mode="subtract_mean")
    assert_same_result(got.detections, exp["result"], "subtract-mean mode")
    # test_pipeline.cpp:344-354 uses a 64 x 64 zero frame at prf 68.6: with 64
    # traces the bin spacing is 1.07 Hz and the reference itself throws from
    # band_select; the drop-in must throw the same error. The property is then
    # checked on a frame long enough to resolve the band.
    from oracle.pyoracle import OracleError
    z = np.zeros((64, 64))
    with pytest.raises(OracleError) as re:
        ref.detect(z, guard_radius=1, background_radius=2)
    with pytest.raises(uwb.ConfigurationError) as ge:
        uwb.detect(F(uwb, z), uwb.PipelineConfig(cfar=uwb.CfarParams(1, 2)))
    assert str(ge.value) == re.value.message
    got, exp = _detect_both(uwb, ref, np.zeros((64, 600)), guard_radius=1, background_radius=2)
    assert len(got.detections.detections) == 0 and (got.band_map.power == 0).all()


def test_detect_errors_match_reference(uwb, ref, cuda):  # test_pipeline.cpp:414-438
    from oracle.pyoracle import OracleError
    data, _ = ref.generate_scene(n_traces=64)
    nan = data.copy()
    nan[3, 3] = np.nan
    cases = [
        (data, 68.6, dict(fft_length=32)),
        (data, 68.6, dict(band_low_hz=0.001, band_high_hz=0.002)),
        (uniform_frame(16, 16, 5), 68.6, dict(band_low_hz=30.0, band_high_hz=40.0)),
        (data, 68.6, dict(mean_filter_window=4)),
        (data, 68.6, dict(mean_filter_window=65)),
        (nan, 68.6, dict(mean_filter_window=4)),
        (data[:1], 68.6, {}),
        (data, -1.0, {}),
        (data[:4, :4], 68.6, dict(guard_radius=4, background_radius=1, band_low_hz=1.0, band_high_hz=30.0)),
    ]
    for d, prf, cfg in cases:
        with pytest.raises(OracleError) as re:
            ref.detect(d, prf=prf, **cfg)
        cfg = dict(cfg)
        params = uwb.CfarParams(cfg.pop("guard_radius", 4), cfg.pop("background_radius", 8))
        with pytest.raises(uwb.Error) as ge:
            uwb.detect(F(uwb, d, prf=prf), uwb.PipelineConfig(cfar=params, **cfg))
        assert type(ge.value).__name__ == re.value.kind, cfg
        assert str(ge.value) == re.value.message


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_detect_batch_matches_reference_per_record(uwb, ref, cuda, dtype):
    """Batched device detect: every record's band map and CFAR
    result equal the reference detect() on that record, bit for bit."""
    import torch
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import DetectBatch
    n_rec = 5
    recs = torch.stack([synth.cfg2_record(seed=40 + i, device="cuda") for i in range(n_rec)])
    recs = recs.to(getattr(torch, dtype)).contiguous()
    config = uwb.PipelineConfig(mean_filter_window=5, fft_length=1024, band_low_hz=0.3, band_high_hz=0.8,
                                cfar=uwb.CfarParams(1, 4, 1e-3))
    db = DetectBatch(n_rec, 512, 1024, config, prf=20.0, dtype=recs.dtype, det_capacity=4096)
    assert db.kept == 25
    db(recs)
    torch.cuda.synchronize()
    db.check_inputs()
    host = recs.double().cpu().numpy()
    for i in range(n_rec):
        exp = ref.detect(host[i], prf=20.0, mean_filter_window=5, fft_length=1024, guard_radius=1,
                         background_radius=4, pfa=1e-3)
        assert_bitwise(db.band[i].cpu().numpy(), exp["band_power"], f"record {i} band map")
        assert np.array_equal(db.mask(i), exp["result"].mask), f"record {i} mask"
        d = db.detections(i)
        e = exp["result"].detections
        assert len(d) == len(e)
        assert np.array_equal(d["row"], e["row"]) and np.array_equal(d["col"], e["col"])
        assert_bitwise(d["threshold"], e["threshold"], f"record {i} detection thresholds")


def test_detect_batch_reports_nonfinite_record(uwb, cuda):
    import torch
    from paper_2012_11077_b200.batch import DetectBatch
    recs = torch.randn((3, 64, 128), device="cuda", dtype=torch.float64)
    recs[1, 5, 7] = float("nan")
    config = uwb.PipelineConfig(fft_length=128, band_low_hz=0.3, band_high_hz=0.8, cfar=uwb.CfarParams(1, 2, 1e-3))
    db = DetectBatch(3, 64, 128, config, prf=20.0, dtype=torch.float64)
    db(recs)
    torch.cuda.synchronize()
    fb = db.first_bad.cpu().numpy().astype(np.uint64)
    assert fb[1, 0] == 5 * 128 + 7
    assert fb[0, 0] == np.uint64(0xFFFFFFFFFFFFFFFF) and fb[2, 0] == np.uint64(0xFFFFFFFFFFFFFFFF)
    with pytest.raises(uwb.InputError):
        db.check_inputs()


@pytest.mark.parametrize("m,n,window,band,dtype", [
    (512, 1024, 5, (0.3, 0.8), "float32"),     # config 2
    (3, 1024, 5, (0.3, 0.8), "float64"),       # fewest rows the fused path takes
    (40, 600, 7, (0.3, 0.8), "float32"),       # zero padding to L = 1024
    (37, 1000, 1, (0.3, 0.8), "float64"),      # window 1 = identity
    (64, 1024, 3, (2.0, 9.9), "float32"),      # wide band: bins 102..506 (most butterflies needed)
    (16, 1024, 9, (9.95, 9.99), "float64"),    # band at the top of the spectrum (bins 509..511)
])
def test_fused_front_end_matches_reference(uwb, ref, cuda, m, n, window, band, dtype):
    """The fused L = 1024 front end (column statistics + one-warp-per-row FFT,
    csrc/frontend.cu) against the reference detect() per record, bit for bit,
    and against the general kernels (flags bit 8)."""
    import torch
    from paper_2012_11077_b200.batch import DetectBatch
    g = torch.Generator(device="cuda").manual_seed(m * 1000 + n)
    recs = torch.randn((3, m, n), device="cuda", dtype=torch.float64, generator=g)
    recs += torch.linspace(-1, 1, n, device="cuda", dtype=torch.float64)[None, None, :] * 0.3
    recs += torch.sin(torch.arange(n, device="cuda", dtype=torch.float64) * 0.13)[None, None, :]
    recs = recs.to(getattr(torch, dtype)).contiguous()
    cfar = uwb.CfarParams(1, 1, 1e-2)
    config = uwb.PipelineConfig(mean_filter_window=window, fft_length=1024, band_low_hz=band[0],
                                band_high_hz=band[1], cfar=cfar)
    outs = []
    for general in (False, True):
        db = DetectBatch(3, m, n, config, prf=20.0, dtype=recs.dtype, det_capacity=1 << 14)
        db(recs, general_kernels=general)
        torch.cuda.synchronize()
        db.check_inputs()
        outs.append((db.band.cpu().numpy().copy(), [db.mask(i) for i in range(3)]))
    assert_bitwise(outs[0][0], outs[1][0], "fused vs general band maps")
    host = recs.double().cpu().numpy()
    for i in range(3):
        exp = ref.detect(host[i], prf=20.0, mean_filter_window=window, fft_length=1024, band_low_hz=band[0],
                         band_high_hz=band[1], guard_radius=1, background_radius=1, pfa=1e-2)
        assert_bitwise(outs[0][0][i], exp["band_power"], f"record {i} band map")
        assert np.array_equal(outs[0][1][i], exp["result"].mask), f"record {i} mask"


def test_fused_front_end_reports_nonfinite(uwb, cuda):
    import torch
    from paper_2012_11077_b200.batch import DetectBatch
    recs = torch.randn((3, 64, 1024), device="cuda", dtype=torch.float32)
    recs[2, 9, 1000] = float("inf")
    recs[2, 30, 3] = float("nan")
    config = uwb.PipelineConfig(fft_length=1024, band_low_hz=0.3, band_high_hz=0.8, cfar=uwb.CfarParams(1, 2, 1e-3))
    db = DetectBatch(3, 64, 1024, config, prf=20.0, dtype=torch.float32)
    db(recs)
    torch.cuda.synchronize()
    fb = db.first_bad.cpu().numpy().astype(np.uint64)
    assert fb[2, 0] == 9 * 1024 + 1000
    assert fb[0, 0] == np.uint64(0xFFFFFFFFFFFFFFFF) and fb[1, 0] == np.uint64(0xFFFFFFFFFFFFFFFF)
    with pytest.raises(uwb.InputError):
        db.check_inputs()
