"""GPU parity: SAT and CA-CFAR through the C ABI vs the reference compiled from
/root/reference (oracle/_ref) and the C restatement. Cases follow the reference's
own tests (proj/tests/test_sat.cpp, test_cfar.cpp); the bar is bit-identity."""
import numpy as np
import pytest

from tests.helpers import (assert_bitwise, assert_same_result, exponential_map, integer_map)

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------------ SAT ---

def test_sat_single_cell(uwb, cuda):  # test_sat.cpp:26-31
    sat = uwb.build_sat(np.array([[7.0]]))
    assert sat.table()[1, 1] == 7.0
    assert sat.region_sum(0, 0, 0, 0) == 7.0


def test_sat_ones_closed_form(uwb, cuda):  # test_sat.cpp:33-43
    sat = uwb.build_sat(np.ones((3, 3)))
    for x in range(3):
        for y in range(3):
            assert sat.table()[x + 1, y + 1] == (x + 1) * (y + 1)


@pytest.mark.parametrize("shape,seed", [((5, 7), 11), ((8, 8), 42), ((16, 16), 7), ((12, 10), 5),
                                        ((1, 1), 1), ((1, 1500), 2), ((1500, 1), 3), ((257, 513), 4),
                                        ((33, 1029), 5), ((64, 2100), 6), ((3, 4097), 7)])
def test_sat_bit_identical_to_reference(uwb, ref, cuda, shape, seed):
    m = np.random.default_rng(seed).uniform(-1, 1, shape)
    got = uwb.build_sat(m).table()
    assert_bitwise(got, ref.build_sat(m), f"SAT {shape}")
    assert (got[0] == 0).all() and (got[:, 0] == 0).all()


def test_sat_fp32_widened_values(uwb, ref, cuda):
    m = np.random.default_rng(9).exponential(1, (300, 700)).astype(np.float32).astype(np.float64)
    assert_bitwise(uwb.build_sat(m).table(), ref.build_sat(m), "SAT fp32-valued")


def test_sat_integer_exact_and_rectangles(uwb, cuda):  # test_sat.cpp:95-109
    rng = np.random.default_rng(5)
    m = rng.integers(0, 1001, (12, 10)).astype(np.float64)
    sat = uwb.build_sat(m)
    for _ in range(100):
        r0, r1 = sorted(rng.integers(0, 12, 2))
        c0, c1 = sorted(rng.integers(0, 10, 2))
        assert sat.region_sum(r0, r1, c0, c1) == m[r0:r1 + 1, c0:c1 + 1].sum()


def test_sat_deterministic(uwb, cuda):  # test_sat.cpp:141-146
    m = np.random.default_rng(77).uniform(0, 1, (15, 31))
    assert_bitwise(uwb.build_sat(m).table(), uwb.build_sat(m).table(), "determinism")


def test_sat_errors(uwb, ref, cuda):  # test_sat.cpp:148-163
    with pytest.raises(uwb.DimensionError):
        uwb.build_sat(np.zeros((0, 4)))
    bad = np.ones((2, 2))
    bad[1, 0] = np.nan
    with pytest.raises(uwb.InputError) as e:
        uwb.build_sat(bad)
    assert str(e.value) == "build_sat: non-finite entry at (1, 0)"
    bad[1, 0] = np.inf
    bad[0, 1] = -np.inf
    with pytest.raises(uwb.InputError) as e:
        uwb.build_sat(bad)
    assert str(e.value) == "build_sat: non-finite entry at (0, 1)"  # first in row-major order
    sat = uwb.build_sat(np.ones((4, 5)))
    for args in [(2, 1, 0, 0), (0, 0, 3, 2), (0, 4, 0, 0), (0, 0, 0, 5)]:
        with pytest.raises(uwb.BoundsError):
            sat.region_sum(*args)


# ----------------------------------------------------------------- CFAR ---

def P(uwb, g, b, pfa):
    return uwb.CfarParams(guard_radius=g, background_radius=b, pfa=pfa)


def test_all_zero_map(uwb, ref, cuda):  # test_cfar.cpp:128-137
    for fn in (uwb.cfar2d_naive, uwb.cfar2d_integral):
        r = fn(np.zeros((32, 32)), uwb.CfarParams())
        assert len(r.detections) == 0 and (r.threshold_map == 0).all() and (r.mask == 0).all()


def test_constant_map(uwb, cuda):  # test_cfar.cpp:139-157
    p = P(uwb, 1, 2, 1e-3)
    for fn in (uwb.cfar2d_naive, uwb.cfar2d_integral):
        assert len(fn(np.full((32, 32), 3.25), p).detections) == 0


def test_exact_tie_is_absent(uwb, cuda):  # test_cfar.cpp:159-170
    r = uwb.cfar2d_naive(np.full((1, 2), 5.0), P(uwb, 0, 1, 0.5))
    assert r.threshold_map[0, 0] == 5.0 and len(r.detections) == 0
    r = uwb.cfar2d_integral(np.full((1, 2), 5.0), P(uwb, 0, 1, 0.5))
    assert r.threshold_map[0, 0] == 5.0 and len(r.detections) == 0


def test_false_alarm_rate(uwb, cuda):  # test_cfar.cpp:172-188
    p = P(uwb, 2, 4, 0.01)
    alarms = cells = 0
    for t in range(100):
        m = exponential_map(64, 64, 1000 + t)
        alarms += len(uwb.cfar2d_integral(m, p).detections)
        cells += m.size
    assert 0.007 < alarms / cells < 0.013


@pytest.mark.parametrize("g,b", [(4, 8), (4, 12), (8, 8), (8, 12)])
def test_integer_maps_bit_identical(uwb, ref, cuda, g, b):  # test_cfar.cpp:190-202
    m = integer_map(48, 48, g * 100 + b)
    p = P(uwb, g, b, 1e-3)
    naive = uwb.cfar2d_naive(m, p)
    integral = uwb.cfar2d_integral(m, p)
    assert np.array_equal(naive.mask, integral.mask)
    assert_bitwise(naive.threshold_map, integral.threshold_map, "naive vs integral on integers")
    assert_same_result(integral, ref.cfar2d(m, g, b, 1e-3, "integral"), "integral vs ref")
    assert_same_result(naive, ref.cfar2d(m, g, b, 1e-3, "naive"), "naive vs ref")


def test_random_float_maps_bit_identical_to_reference(uwb, ref, cuda):  # test_cfar.cpp:204-224
    rng = np.random.default_rng(2024)
    for k in range(40):
        g, b = int(rng.integers(0, 4)), int(rng.integers(1, 5))
        pfa = float(10 ** rng.uniform(-4, -1))
        rows, cols = (int(v) for v in rng.integers(8, 129, 2))
        if rows <= 2 * g + 1 and cols <= 2 * g + 1:
            continue
        m = exponential_map(rows, cols, 5000 + k)
        p = P(uwb, g, b, pfa)
        assert_same_result(uwb.cfar2d_integral(m, p), ref.cfar2d(m, g, b, pfa, "integral"), f"case {k}")
        assert_same_result(uwb.cfar2d_naive(m, p), ref.cfar2d(m, g, b, pfa, "naive"), f"naive case {k}")


def test_pfa_monotone(uwb, cuda):  # test_cfar.cpp:226-239
    m = exponential_map(48, 48, 321)
    strict = uwb.cfar2d_integral(m, P(uwb, 2, 4, 1e-3))
    loose = uwb.cfar2d_integral(m, P(uwb, 2, 4, 1e-2))
    assert (loose.mask >= strict.mask).all()


def test_scale_covariance(uwb, cuda):  # test_cfar.cpp:241-276
    m = exponential_map(40, 40, 654)
    p = P(uwb, 1, 3, 1e-3)
    for fn in (uwb.cfar2d_naive, uwb.cfar2d_integral):
        base = fn(m, p)
        for k in (4.0, 0.25):
            big = fn(m * k, p)
            assert np.array_equal(base.mask, big.mask)
            assert_bitwise(big.threshold_map, base.threshold_map * k, "power-of-two scale")
    base = uwb.cfar2d_integral(m, p)
    big = uwb.cfar2d_integral(m * 3.7, p)
    assert np.array_equal(base.mask, big.mask)
    np.testing.assert_allclose(big.threshold_map, base.threshold_map * 3.7, rtol=1e-12)


def test_detection_list_is_mask_sorted(uwb, cuda):  # test_cfar.cpp:278-306
    m = exponential_map(32, 32, 888)
    r = uwb.cfar2d_integral(m, P(uwb, 1, 2, 0.05))
    d = r.detections
    assert len(d) == r.mask.sum() > 0
    assert (r.mask[d["row"].astype(int), d["col"].astype(int)] == 1).all()
    assert (d["value"] == m[d["row"].astype(int), d["col"].astype(int)]).all()
    assert (d["value"] > d["threshold"]).all()
    assert (np.diff(d["value"]) <= 0).all()
    assert np.array_equal(m > r.threshold_map, r.mask == 1)


def test_threads_argument_ignored(uwb, cuda):  # test_cfar.cpp:308-320
    m = exponential_map(60, 45, 4242)
    p = P(uwb, 2, 3, 1e-3)
    for fn in (uwb.cfar2d_naive, uwb.cfar2d_integral):
        assert_same_result(fn(m, p, 1), fn(m, p, 4), "threads")


def test_input_validation_and_messages(uwb, ref, cuda):  # test_cfar.cpp:322-347
    from oracle.pyoracle import OracleError
    cases = []
    neg = np.ones((16, 16)); neg[3, 4] = -0.5
    cases.append(("naive", neg, 4, 8, 1e-3))
    cases.append(("integral", neg, 4, 8, 1e-3))
    nan = np.ones((20, 20)); nan[0, 0] = np.nan
    cases.append(("integral", nan, 4, 8, 1e-3))
    cases.append(("naive", nan, 4, 8, 1e-3))
    cases.append(("integral", nan, -1, 8, 1e-3))   # SAT error wins over parameter error
    cases.append(("naive", nan, -1, 8, 1e-3))      # parameter error first for naive
    cases.append(("naive", np.ones((8, 8)), 4, 8, 1e-3))
    cases.append(("integral", np.ones((8, 8)), 4, 8, 1e-3))
    cases.append(("naive", np.ones((16, 16)), -1, 8, 1e-3))
    cases.append(("naive", np.ones((16, 16)), 1, 0, 1e-3))
    cases.append(("integral", np.ones((16, 16)), 1, 2, 1.5))
    cases.append(("integral", np.zeros((0, 5)), 1, 2, 0.1))
    cases.append(("naive", np.zeros((0, 5)), 1, 2, 0.1))
    for backend, m, g, b, pfa in cases:
        with pytest.raises(OracleError) as re:
            ref.cfar2d(m, g, b, pfa, backend)
        fn = uwb.cfar2d_naive if backend == "naive" else uwb.cfar2d_integral
        with pytest.raises(uwb.Error) as ge:
            fn(m, P(uwb, g, b, pfa))
        assert type(ge.value).__name__ == re.value.kind, (backend, g, b, pfa)
        assert str(ge.value) == re.value.message
    # a map long in one dimension keeps training cells
    uwb.cfar2d_naive(np.ones((8, 64)), P(uwb, 4, 8, 1e-3))


def test_alpha_and_windows_match_reference(uwb, ref, cuda):  # test_cfar.cpp:60-126
    assert uwb.alpha_factor(1, 0.5) == 1.0
    assert abs(uwb.alpha_factor(24, 1e-3) - 8.0045143719197766) <= 1e-12 * 8.0045143719197766
    for n in (1, 4, 24, 416, 544, 5248):
        for pfa in (1e-6, 1e-4, 1e-3, 1e-2, 0.1, 0.5, 0.9):
            assert uwb.alpha_factor(n, pfa) == ref.alpha_factor(n, pfa)
    w = uwb.training_window(P(uwb, 1, 1, 1e-3), 0, 0, 100, 100)
    assert (w.outer.area(), w.guard.area(), w.n_train) == (9, 4, 5)
    assert uwb.training_window(P(uwb, 4, 8, 1e-3), 100, 100, 1024, 600).n_train == 544
