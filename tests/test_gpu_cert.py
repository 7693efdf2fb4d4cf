"""GPU parity of the certified-decision CFAR path (csrc/cfar_cert.cu): the
default path of BatchCfar for mask + list outputs. It must give exactly the
masks, detection lists and counts of the exact two-kernel path (full fp64
table + cfar_ws_kernel, itself bit-identical to cfar2d_integral of
/root/reference/proj/src/cfar.cpp:218-227), report the tie band
(|cut - T| <= 1e-6 T) exactly, and hand maps it cannot certify (values outside
its range, candidate-list overflow) to the exact path inside the same call."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pair(n, rows, cols, p, dtype=torch.float32, **kw):
    from paper_2012_11077_b200.batch import BatchCfar
    cert = BatchCfar(n, rows, cols, p, dtype, **kw)
    exact = BatchCfar(n, rows, cols, p, dtype, **kw)
    return cert, exact


def _same(cert, exact, n, what, expect_status=0):
    st = cert.cert_status.cpu().numpy()
    if expect_status is not None:
        assert (st == expect_status).all(), f"{what}: cert_status {st[:8]}"
    assert torch.equal(cert.counts, exact.counts), f"{what}: counts"
    assert torch.equal(cert.mask_bits, exact.mask_bits), f"{what}: mask bits"
    for i in range(n):
        a, b = cert.detections(i), exact.detections(i)
        assert a.tobytes() == b.tobytes(), f"{what}: map {i} detection list"


def _tie_band_from_thresholds(maps_host, thr):
    """Cells with |cut - T| <= 1e-6 T from the exact threshold map."""
    cut = maps_host.astype(np.float64)
    return np.argwhere(np.abs(cut - thr) <= 1e-6 * thr)


def test_cfg3_shape_certified_equals_exact_and_reference(uwb, ref, cuda):
    from paper_2012_11077_b200 import synth
    n = 24
    maps = synth.cfg3_maps(n, seed=11, device=cuda)
    p = uwb.CfarParams(2, 8, 1e-4)
    cert, exact = _pair(n, 1024, 1024, p, det_capacity=1024)
    cert(maps, certify=True)
    exact(maps, exact=True)
    torch.cuda.synchronize()
    cert.check_inputs()
    _same(cert, exact, n, "cfg3")
    assert (exact.cert_status.cpu().numpy() == -1).all()  # the exact call reports "not certified"
    host = maps.double().cpu().numpy()
    for i in (0, 7, n - 1):
        r = ref.cfar2d(host[i], 2, 8, 1e-4, "integral")
        assert np.array_equal(cert.mask(i), r.mask), f"map {i} mask vs reference"
        d, e = cert.detections(i), r.detections
        assert len(d) == len(e) and np.array_equal(d["row"], e["row"]) and np.array_equal(d["col"], e["col"])
        assert np.array_equal(d["threshold"].view(np.uint64), np.asarray(e["threshold"]).view(np.uint64))

def test_tie_band_matches_exact_thresholds(uwb, cuda):
    """Cells placed at T(1 + d) for d in {0, +-4e-7, +-3e-6, 1e-9} (their own T
    does not depend on them: the CUT is inside its guard window): the certified
    path must list exactly the cells with |cut - T| <= 1e-6 T of the exact
    threshold map, with T bit-identical, and decide them like the exact path."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    n, R, C = 2, 512, 512
    maps = synth.exponential_maps(n, R, C, seed=5, dtype=torch.float64, device=cuda)
    p = uwb.CfarParams(2, 8, 1e-3)
    full = BatchCfar(n, R, C, p, torch.float64, det_capacity=4096, want_thresholds=True)
    full(maps)
    torch.cuda.synchronize()
    thr = full.thresholds.clone()
    deltas = torch.tensor([0.0, 4e-7, -4e-7, 3e-6, -3e-6, 1e-9], dtype=torch.float64, device=cuda)
    rr, cc = torch.meshgrid(torch.arange(15, R - 15, 30, device=cuda), torch.arange(15, C - 15, 30, device=cuda),
                            indexing="ij")
    rr, cc = rr.reshape(-1), cc.reshape(-1)
    d = deltas[torch.arange(rr.numel(), device=cuda) % deltas.numel()]
    for i in range(n):
        maps[i, rr, cc] = thr[i, rr, cc] * (1.0 + d)
    full(maps)
    cert = BatchCfar(n, R, C, p, torch.float64, det_capacity=4096, tie_capacity=4096)
    cert(maps, certify=True)
    torch.cuda.synchronize()
    # placed cells keep their T up to the table rounding (every cell enters every later table entry)
    assert torch.allclose(full.thresholds[:, rr, cc], thr[:, rr, cc], rtol=1e-9, atol=0)
    assert (cert.cert_status.cpu().numpy() == 0).all()
    host = maps.cpu().numpy()
    for i in range(n):
        t2 = full.thresholds[i].cpu().numpy()
        assert np.array_equal(cert.mask(i), full.mask(i)), f"map {i} mask"
        assert cert.detections(i).tobytes() == full.detections(i).tobytes(), f"map {i} detections"
        want = _tie_band_from_thresholds(host[i], t2)
        got = cert.tie_band(i)
        assert len(want) >= 3 * rr.numel() // 6, f"map {i}: only {len(want)} tie cells"
        assert len(got) == len(want), f"map {i}: {len(got)} vs {len(want)} tie cells"
        assert np.array_equal(got["row"], want[:, 0]) and np.array_equal(got["col"], want[:, 1])
        assert np.array_equal(got["threshold"].view(np.uint64), t2[want[:, 0], want[:, 1]].view(np.uint64))


@pytest.mark.parametrize("shape", [
    ((1, 1, 4, 4), 1e-3, (6, 512, 26), torch.float64),   # config 2-like band maps (even width)
    ((2, 2, 8, 8), 1e-4, (2, 256, 512), torch.float64),  # config 1
    ((1, 3, 4, 16), 1e-3, (3, 700, 600), torch.float32),  # config 5 windows
    ((3, 1, 16, 4), 1e-5, (3, 700, 600), torch.float32),
    ((4, 4, 32, 32), 1e-5, (1, 1100, 900), torch.float32),  # config 4 window
], ids=["cfg2", "cfg1", "cfg5a", "cfg5b", "cfg4"])
def test_instantiated_windows_equal_exact(uwb, cuda, shape):
    (gr, gc, br, bc), pfa, (n, R, C), dt = shape
    from paper_2012_11077_b200 import synth
    maps = synth.cfg5_maps(n, seed=21, device=cuda, rows=R, cols=C).to(dt) if C >= 64 else \
        synth.exponential_maps(n, R, C, seed=21, dtype=dt, device=cuda)
    synth.add_point_targets(maps, 5, 10.0, 20.0, seed=22)
    p = uwb.CfarParams(guard_radius=gr, background_radius=br, pfa=pfa, guard_cols=gc, background_cols=bc)
    cert, exact = _pair(n, R, C, p, dt, det_capacity=1 << 14)
    cert(maps, certify=True)
    exact(maps, exact=True)
    torch.cuda.synchronize()
    _same(cert, exact, n, f"window {(gr, gc, br, bc)}")


def test_out_of_range_and_overflow_maps_run_exact(uwb, cuda):
    """Map 1 holds a value >= 2^9 (outside the certified range), map 2 is all
    zeros (every cell a candidate: list overflow); both run the exact path in
    the same call, the others stay certified, and all outputs equal the exact path."""
    from paper_2012_11077_b200 import synth
    n = 4
    maps = synth.cfg3_maps(n, seed=31, device=cuda)
    maps[1, 500, 600] = 1000.0
    maps[2].zero_()
    p = uwb.CfarParams(2, 8, 1e-4)
    cert, exact = _pair(n, 1024, 1024, p, det_capacity=2048)
    cert(maps, certify=True)
    exact(maps, exact=True)
    torch.cuda.synchronize()
    st = cert.cert_status.cpu().numpy()
    assert st[0] == 0 and st[3] == 0 and (st[1] & 2) and (st[2] & 1), st
    _same(cert, exact, n, "fallback", expect_status=None)
    assert cert.tie_counts[1].item() == -1 and cert.tie_counts[2].item() == -1


def test_input_errors_reported_like_exact_path(uwb, cuda):
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.errors import InputError
    n = 3
    maps = synth.cfg3_maps(n, seed=41, device=cuda)
    maps[0, 10, 20] = float("nan")
    maps[0, 5, 900] = -1.0    # the non-finite cell wins (build_sat runs first, cfar.cpp:218-227)
    maps[1, 700, 3] = -0.5
    maps[2, 0, 0] = -0.0      # a valid zero
    p = uwb.CfarParams(2, 8, 1e-4)
    cert, exact = _pair(n, 1024, 1024, p, det_capacity=1024)
    cert(maps, certify=True)
    exact(maps, exact=True)
    torch.cuda.synchronize()
    assert torch.equal(cert.first_bad, exact.first_bad)
    fb = cert.first_bad.cpu().numpy()
    assert fb[0, 0] == 10 * 1024 + 20 and fb[1, 1] == 700 * 1024 + 3 and fb[2, 0] == -1 and fb[2, 1] == -1
    with pytest.raises(InputError, match="non-finite"):
        cert.check_inputs()
    assert cert.detections(2).tobytes() == exact.detections(2).tobytes()


def test_row_window_tiles_equal_exact(uwb, cuda):
    """Config 4 path: a rank's row window with column-band tables (tile-local
    taps) equals the exact tile path cell for cell."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    R, C = 3000, 2048
    full = synth.cfg4_map(seed=51, device=cuda, rows=R, cols=C)
    p = uwb.CfarParams(4, 32, 1e-5)
    for (r0, r1) in [(0, 1100), (1100, 3000)]:
        b0, b1 = max(0, r0 - 36), min(R, r1 + 36)
        buf = full[b0:b1].contiguous().unsqueeze(0)
        win = (R, b0, r0, r1, 1024)
        cert = BatchCfar(1, b1 - b0, C, p, torch.float32, det_capacity=1 << 15, window=win, slab_rows=512)
        exact = BatchCfar(1, b1 - b0, C, p, torch.float32, det_capacity=1 << 15, window=win, slab_rows=512)
        cert(buf, certify=True)
        exact(buf, exact=True)
        torch.cuda.synchronize()
        _same(cert, exact, 1, f"rows [{r0}, {r1})")


def test_odd_width_runs_exact_path(uwb, cuda):
    """Maps with an odd column count (config 2's 25-bin band) take the exact path."""
    from paper_2012_11077_b200 import synth
    maps = synth.exponential_maps(3, 512, 25, seed=61, dtype=torch.float64, device=cuda)
    p = uwb.CfarParams(1, 4, 1e-3)
    cert, exact = _pair(3, 512, 25, p, torch.float64, det_capacity=1024)
    cert(maps, certify=True)
    exact(maps, exact=True)
    torch.cuda.synchronize()
    _same(cert, exact, 3, "odd width", expect_status=-1)


def test_large_batch_with_fallback_maps_equals_exact(uwb, cuda):
    """A 1200-map batch gives exactly the exact path's results, with a map the
    certificate cannot cover (a value >= 2^9: exact fallback inside the same
    call) in the middle of the batch, and reports a non-finite cell of a later
    map as the reference's InputError."""
    from paper_2012_11077_b200 import synth
    n, R, C = 1200, 256, 1024
    gen = torch.Generator(device="cuda").manual_seed(77)
    maps = torch.empty((n, R, C), device=cuda, dtype=torch.float32).exponential_(1.0, generator=gen)
    maps[:, 100, 500] += 40.0
    maps[700, 10, 10] = 1000.0        # outside the certified range: exact fallback for map 700
    p = uwb.CfarParams(2, 8, 1e-4)
    cert, exact = _pair(n, R, C, p, det_capacity=256)
    cert(maps, certify=True)
    exact(maps, exact=True)
    torch.cuda.synchronize()
    st = cert.cert_status.cpu().numpy()
    assert st[700] != 0 and (np.delete(st, 700) == 0).all()
    _same(cert, exact, n, "large batch", expect_status=None)
    maps[1100, 3, 4] = float("nan")
    cert(maps, certify=True)
    torch.cuda.synchronize()
    fb = cert.first_bad.cpu().numpy().astype(np.uint64)
    assert fb[1100, 0] == 3 * C + 4
    with pytest.raises(uwb.InputError):
        cert.check_inputs()
