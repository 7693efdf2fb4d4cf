"""CPU: pin the oracle. The plain-C restatement (oracle/uwb_oracle.c) must be
bit-identical to the reference compiled from /root/reference (oracle/_ref), and
both must pass the reference tests' known-answer values (proj/tests/*.cpp) and
the committed golden fixtures (tests/golden/, generated from the reference by
tests/golden/make_golden.py)."""
import math
import os

import numpy as np
import pytest

from tests.helpers import assert_bitwise, exponential_map, integer_map, uniform_frame

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------- KATs (reference tests) ---

def test_alpha_kats(ref, oracle):  # test_cfar.cpp:60-81
    for lib in (ref.alpha_factor, oracle.alpha):
        assert lib(1, 0.5) == 1.0
        assert abs(lib(24, 1e-3) - 8.0045143719197766) <= 1e-12 * 8.0045143719197766
        for n in (1, 4, 24, 544):
            prev = math.inf
            for pfa in (1e-6, 1e-4, 1e-3, 1e-2, 0.1, 0.5, 0.9):
                a = lib(n, pfa)
                assert 0 < a < prev
                prev = a
    for n in range(1, 600):
        assert ref.alpha_factor(n, 1e-4) == oracle.alpha(n, 1e-4)


def test_training_window_kats(ref, oracle):  # test_cfar.cpp:90-126
    w = ref.training_window(1, 1, 1e-3, 50, 50, 100, 100)
    assert w["n_train"] == 16
    w = ref.training_window(1, 1, 1e-3, 0, 0, 100, 100)
    assert w["n_train"] == 5
    assert ref.training_window(4, 8, 1e-3, 100, 100, 1024, 600)["n_train"] == 544
    assert oracle.interior_train_count(4, 4, 8, 8) == 544
    assert oracle.interior_train_count(2, 2, 8, 8) == 416
    assert oracle.interior_train_count(4, 4, 32, 32) == 5248
    assert oracle.interior_train_count(1, 3, 4, 16) == 408


def test_sat_kats(ref, oracle):  # test_sat.cpp:26-58
    for lib in (ref.build_sat, oracle.build_sat):
        t = lib(np.array([[7.0]]))
        assert t[1, 1] == 7.0
        t = lib(np.ones((3, 3)))
        assert all(t[x + 1, y + 1] == (x + 1) * (y + 1) for x in range(3) for y in range(3))
        t = lib(np.random.default_rng(11).uniform(0, 1, (5, 7)))
        assert (t[0] == 0).all() and (t[:, 0] == 0).all()


def test_cfar_kats(ref, oracle):  # test_cfar.cpp:128-170
    z = ref.cfar2d(np.zeros((32, 32)), 4, 8, 1e-3)
    assert len(z.detections) == 0 and (z.threshold_map == 0).all()
    r = ref.cfar2d(np.full((1, 2), 5.0), 0, 1, 0.5, "naive")
    assert r.threshold_map[0, 0] == 5.0 and len(r.detections) == 0
    o = oracle.cfar(np.full((1, 2), 5.0), 0, 0, 1, 1, 0.5, "naive")
    assert o.threshold_map[0, 0] == 5.0 and len(o.detections) == 0


# ----------------------------------------- restatement == reference bitwise ---

def test_restatement_sat_bitwise(ref, oracle):
    rng = np.random.default_rng(1)
    for k in range(20):
        shape = tuple(int(v) for v in rng.integers(1, 70, 2))
        m = rng.uniform(-1, 1, shape)
        assert_bitwise(oracle.build_sat(m), ref.build_sat(m), f"SAT {shape}")


def test_restatement_cfar_bitwise(ref, oracle):
    rng = np.random.default_rng(7)
    for k in range(30):
        g, b = int(rng.integers(0, 4)), int(rng.integers(1, 6))
        rows, cols = (int(v) for v in rng.integers(8, 90, 2))
        if rows <= 2 * g + 1 and cols <= 2 * g + 1:
            continue
        pfa = float(10 ** rng.uniform(-4, -1))
        m = exponential_map(rows, cols, k) if k % 3 else integer_map(rows, cols, k)
        for backend in ("integral", "naive"):
            a = ref.cfar2d(m, g, b, pfa, backend)
            o = oracle.cfar(m, g, g, b, b, pfa, backend)
            assert np.array_equal(a.mask, o.mask)
            assert_bitwise(a.threshold_map, o.threshold_map, f"{backend} case {k}")
            assert np.array_equal(a.detections, o.detections)


def test_restatement_errors_match_reference(ref, oracle):
    from oracle.pyoracle import OracleError
    neg = np.ones((16, 16))
    neg[3, 4] = -0.5
    nan = np.ones((20, 20))
    nan[0, 0] = np.nan
    for m, g, b, pfa, backend in [(neg, 4, 8, 1e-3, "naive"), (nan, 4, 8, 1e-3, "integral"),
                                  (nan, -1, 8, 1e-3, "integral"), (nan, -1, 8, 1e-3, "naive"),
                                  (np.ones((8, 8)), 4, 8, 1e-3, "integral"), (np.ones((16, 16)), 1, 0, 0.1, "naive")]:
        with pytest.raises(OracleError) as e1:
            ref.cfar2d(m, g, b, pfa, backend)
        with pytest.raises(OracleError) as e2:
            oracle.cfar(m, g, g, b, b, pfa, backend)
        assert e1.value.code == e2.value.code


def test_restatement_frontend_bitwise(ref, oracle):
    for shape, seed in [((128, 24), 9), ((64, 100), 3), ((7, 33), 5)]:
        d = uniform_frame(*shape, seed)
        for op in ("remove_dc", "detrend_linear", "subtract_slow_time_mean"):
            assert_bitwise(oracle.frame_stage(op, d), ref.frame_stage(op, d), op)
        assert_bitwise(oracle.frame_stage("mean_filter_slow", d, 5), ref.frame_stage("mean_filter_slow", d, 5), "mf")
        assert_bitwise(oracle.frame_stage("normalize_slow", d, 1, 1e-12),
                       ref.frame_stage("normalize_slow", d, 1, 1e-12), "norm")
        for L in (shape[1], 1 << (shape[1] - 1).bit_length(), 2 * shape[1] + 3):
            assert_bitwise(oracle.slow_time_spectrum(d, L), ref.slow_time_spectrum(d, L)[0], f"spectrum L={L}")


def test_restatement_detect_bitwise(ref, oracle):
    data, truth = ref.generate_scene(seed=7)
    a = ref.detect(data)
    o = oracle.detect(data, guard_rows=4, background_rows=8)
    assert_bitwise(o["band_power"], a["band_power"], "band")
    assert np.array_equal(o["result"].mask, a["result"].mask)
    assert np.array_equal(o["result"].detections, a["result"].detections)


# ------------------------------------------- FFT provider vs FFTW's contract ---

def test_fft_provider_reference_tests(ref):  # test_pipeline.cpp:202-275
    n, k0 = 64, 9
    v = np.cos(2 * math.pi * k0 * np.arange(n) / n)
    p, _, _ = ref.slow_time_spectrum(np.vstack([v, v]), n, prf=64.0)
    expect = (n / 2) ** 2
    assert abs(p[0, k0] - expect) <= 1e-9 * expect
    assert (np.delete(p[0], k0) <= 1e-9 * expect).all()
    p, _, _ = ref.slow_time_spectrum(np.zeros((3, 20)), 32)
    assert (p == 0).all()
    d = uniform_frame(2, 50, 71)
    p, _, _ = ref.slow_time_spectrum(d, 64)
    for r in range(2):
        x = np.zeros(64)
        x[:50] = d[r]
        X = np.array([sum(x[j] * complex(math.cos(-2 * math.pi * k * j / 64), math.sin(-2 * math.pi * k * j / 64))
                          for j in range(64)) for k in range(64)])
        assert abs((np.abs(X) ** 2).sum() - 64 * (d[r] ** 2).sum()) <= 1e-9 * 64 * (d[r] ** 2).sum()
        np.testing.assert_allclose(p[r], np.abs(X[:33]) ** 2, rtol=1e-9, atol=0)
    p, f, _ = ref.slow_time_spectrum(uniform_frame(4, 600, 15), 1024, prf=68.6)
    bp, bf = ref.band_select(p, f, 0.3, 0.8)
    assert bf.size == 7 and bf[0] == f[5] and bf[-1] == f[11]


def test_fft_provider_matches_numpy(ref):
    for n, L in [(1000, 1024), (600, 600), (333, 512)]:
        d = uniform_frame(3, n, n)
        p, _, _ = ref.slow_time_spectrum(d, L)
        x = np.zeros((3, L))
        x[:, :n] = d
        exact = np.abs(np.fft.rfft(x, axis=1)) ** 2
        scale = np.maximum(exact, 1e-12 * exact.max(axis=1, keepdims=True))
        assert (np.abs(p - exact) / scale).max() < 1e-9


# --------------------------------------------------------- golden fixtures ---

def _golden_files():
    return sorted(f for f in os.listdir(GOLDEN) if f.endswith(".npz")) if os.path.isdir(GOLDEN) else []


@pytest.mark.parametrize("name", _golden_files())
def test_restatement_reproduces_golden(oracle, name):
    g = np.load(os.path.join(GOLDEN, name))
    kind = str(g["kind"])
    if kind == "sat":
        assert_bitwise(oracle.build_sat(g["input"]), g["table"], name)
    elif kind == "cfar":
        p = g["params"]
        r = oracle.cfar(g["input"], int(p[0]), int(p[0]), int(p[1]), int(p[1]), float(p[2]), str(g["backend"]))
        assert np.array_equal(r.mask, g["mask"])
        assert_bitwise(r.threshold_map, g["threshold_map"], name)
        assert_bitwise(r.detections["value"], g["det_value"], name)
        assert np.array_equal(r.detections["row"], g["det_row"]) and np.array_equal(r.detections["col"], g["det_col"])
    elif kind == "spectrum":
        assert_bitwise(oracle.slow_time_spectrum(g["input"], int(g["fft_length"])), g["power"], name)
    elif kind == "detect":
        r = oracle.detect(g["input"], prf=float(g["prf"]), guard_rows=int(g["guard"]),
                          background_rows=int(g["train"]), pfa=float(g["pfa"]))
        assert_bitwise(r["band_power"], g["band_power"], name)
        assert np.array_equal(r["result"].mask, g["mask"])
    else:
        pytest.fail(f"unknown golden kind {kind}")


def test_golden_fixtures_present():
    assert len(_golden_files()) >= 8
