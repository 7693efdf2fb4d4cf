"""The fused SAT+CFAR kernel (csrc/cfar_fused.cu): bit-identical to the
two-kernel path (table in HBM; the fused kernel is flags bit 4) and to the reference / restatement
over band edges, partial bands, every columns-per-lane variant, both ring
occupancies, f32/f64, per-cell outputs, the unit queue wrapping many times,
a single wide map (band chain), and non-finite / negative input reports."""
import numpy as np
import pytest
import torch

from tests.helpers import assert_bitwise

pytestmark = pytest.mark.gpu


def _run(uwb, maps, p, per_cell, fused, cap=1 << 14):
    from paper_2012_11077_b200.batch import BatchCfar, kernel_launches
    n, R, C = maps.shape
    b = BatchCfar(n, R, C, p, maps.dtype, det_capacity=cap, want_mask_u8=per_cell, want_thresholds=per_cell)
    k0 = kernel_launches()
    b(maps, fused=fused, exact=not fused)  # the exact two-kernel path, not the certified one
    torch.cuda.synchronize()
    return b, kernel_launches() - k0


def _same(a, b, what):
    assert torch.equal(a.mask_bits, b.mask_bits), f"{what}: mask bits"
    assert torch.equal(a.counts, b.counts), f"{what}: counts"
    assert torch.equal(a.first_bad, b.first_bad), f"{what}: first_bad"
    if a.thresholds is not None:
        assert torch.equal(a.mask_u8, b.mask_u8), f"{what}: mask"
        assert_bitwise(a.thresholds.cpu().numpy(), b.thresholds.cpu().numpy(), f"{what}: thresholds")
    for i in range(a.n_maps):
        da, db = a.detections(i), b.detections(i)
        assert len(da) == len(db) and da.tobytes() == db.tobytes(), f"{what}: map {i} detections"


CASES = [
    # n, rows, cols, dtype, (guard_r, bg_r, guard_c, bg_c), pfa
    (5, 300, 1000, torch.float32, (2, 8, 2, 8), 1e-3),    # partial last band, hc 10 (5 cols/lane)
    (3, 77, 130, torch.float64, (1, 4, 3, 16), 1e-2),     # f64, hc 19 (6 cols/lane)
    (2, 90, 700, torch.float32, (3, 10, 8, 32), 1e-2),    # hc 40 (8 cols/lane)
    (2, 400, 300, torch.float32, (4, 36, 1, 3), 1e-3),    # hr 40: one CTA per SM ring
    (1, 200, 3000, torch.float32, (2, 8, 2, 8), 1e-3),    # one wide map: 24-band chain
    (600, 40, 256, torch.float32, (1, 3, 1, 3), 1e-2),    # 1200 units: unit queue wraps
    (4, 1, 200, torch.float32, (0, 1, 1, 2), 5e-2),       # one row
    (4, 6, 33, torch.float64, (1, 2, 1, 2), 5e-2),        # tiny
]


@pytest.mark.parametrize("per_cell", [False, True])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_fused_matches_two_kernel_path(uwb, cuda, case, per_cell):
    n, R, C, dt, (gr, br, gc, bc), pfa = CASES[case]
    gen = torch.Generator(device="cuda").manual_seed(100 + case)
    maps = torch.empty((n, R, C), device=cuda, dtype=dt).exponential_(1.0, generator=gen)
    maps[:, ::7, ::5] *= 40.0  # targets
    p = uwb.CfarParams(guard_radius=gr, background_radius=br, pfa=pfa, guard_cols=gc, background_cols=bc)
    fused, k_f = _run(uwb, maps, p, per_cell, fused=True)
    two, k_t = _run(uwb, maps, p, per_cell, fused=False)
    # SAT + CFAR -> one kernel; a wide single map's exact SAT is a chain of clusters,
    # which also launches the fill of its boundary columns
    assert k_f in (k_t - 1, k_t - 2), "the fused call launches fewer kernels (SAT + CFAR -> one)"
    _same(fused, two, f"case {case}")
    assert int(fused.counts.sum()) > 0


@pytest.mark.parametrize("case", [0, 1, 4])
def test_fused_vs_restatement(uwb, oracle, cuda, case):
    n, R, C, dt, (gr, br, gc, bc), pfa = CASES[case]
    gen = torch.Generator(device="cuda").manual_seed(7 + case)
    maps = torch.empty((min(n, 2), R, C), device=cuda, dtype=dt).exponential_(1.0, generator=gen)
    p = uwb.CfarParams(guard_radius=gr, background_radius=br, pfa=pfa, guard_cols=gc, background_cols=bc)
    b, _ = _run(uwb, maps, p, True, fused=True)
    host = maps.double().cpu().numpy()
    for i in range(maps.shape[0]):
        r = oracle.cfar(host[i], gr, gc, br, bc, pfa)
        assert np.array_equal(b.mask_u8[i].cpu().numpy(), r.mask), f"case {case} map {i} mask"
        assert np.array_equal(b.mask(i), r.mask)
        assert_bitwise(b.thresholds[i].cpu().numpy(), r.threshold_map, f"case {case} map {i} thresholds")


def test_fused_cfg3_maps_vs_reference(uwb, ref, cuda):
    """BASELINE config 3 maps, mask-bits-only mode (the interior fast path)."""
    from paper_2012_11077_b200 import synth
    maps = synth.cfg3_maps(4, seed=33, device=cuda)
    p = uwb.CfarParams(2, 8, 1e-4)
    b, _ = _run(uwb, maps, p, False, fused=True, cap=1024)
    host = maps.double().cpu().numpy()
    for i in range(4):
        r = ref.cfar2d(host[i], 2, 8, 1e-4, "integral")
        assert np.array_equal(b.mask(i), r.mask), f"map {i} mask"
        d = b.detections(i)
        assert len(d) == len(r.detections)
        assert np.array_equal(d["row"], r.detections["row"]) and np.array_equal(d["col"], r.detections["col"])
        assert_bitwise(d["threshold"], r.detections["threshold"], f"map {i} det thresholds")


def test_fused_reports_bad_inputs(uwb, cuda):
    """First non-finite input (SAT wavefront) and first negative CUT, row-major,
    exactly as the two-kernel path reports them."""
    gen = torch.Generator(device="cuda").manual_seed(3)
    maps = torch.empty((3, 130, 600), device=cuda).exponential_(1.0, generator=gen)
    maps[0, 100, 590] = float("nan")
    maps[0, 120, 3] = float("inf")
    maps[1, 5, 200] = -1.0
    maps[1, 64, 7] = -2.0
    maps[2, 129, 599] = float("-inf")
    p = uwb.CfarParams(2, 8, 1e-3)
    fused, _ = _run(uwb, maps, p, False, fused=True)
    two, _ = _run(uwb, maps, p, False, fused=False)
    fb = fused.first_bad.cpu().numpy().astype(np.uint64)
    assert int(fb[0, 0]) == 100 * 600 + 590
    assert int(fb[1, 1]) == 5 * 600 + 200
    assert int(fb[2, 0]) == 129 * 600 + 599
    assert torch.equal(fused.first_bad, two.first_bad)
