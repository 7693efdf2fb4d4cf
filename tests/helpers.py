"""Shared comparison helpers for parity tests."""
import numpy as np


def bits(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(a, b, what=""):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape, f"{what}: shape {a.shape} != {b.shape}"
    diff = bits(a) != bits(b)
    if diff.any():
        idx = np.argwhere(diff)[:5]
        raise AssertionError(f"{what}: {int(diff.sum())} of {diff.size} values differ bitwise; first at "
                             f"{idx.tolist()}: {a[tuple(idx[0])]!r} vs {b[tuple(idx[0])]!r}")


def assert_same_result(gpu, ref, what=""):
    """DetectionResult-like (mask, threshold_map, detections) bit-identical."""
    assert np.array_equal(np.asarray(gpu.mask), np.asarray(ref.mask)), f"{what}: mask differs"
    assert_bitwise(gpu.threshold_map, ref.threshold_map, f"{what}: threshold_map")
    gd, rd = gpu.detections, ref.detections
    assert len(gd) == len(rd), f"{what}: {len(gd)} detections vs {len(rd)}"
    for f in ("row", "col"):
        assert np.array_equal(gd[f], rd[f]), f"{what}: detection {f} order differs"
    assert_bitwise(gd["value"], rd["value"], f"{what}: detection values")
    assert_bitwise(gd["threshold"], rd["threshold"], f"{what}: detection thresholds")


def exponential_map(rows, cols, seed):
    return np.random.default_rng(seed).exponential(1.0, (rows, cols))


def integer_map(rows, cols, seed, hi=500):
    return np.random.default_rng(seed).integers(0, hi + 1, (rows, cols)).astype(np.float64)


def uniform_frame(m, n, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, (m, n))
