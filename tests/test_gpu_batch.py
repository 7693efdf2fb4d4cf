"""GPU parity of the batched device path (BatchCfar, the path bench.py times)
against the reference (square windows) and the C restatement (per-axis windows,
row-slab tables), on inputs from the BASELINE.json config generators."""
import numpy as np
import pytest
import torch

from tests.helpers import assert_bitwise

pytestmark = pytest.mark.gpu


def _check_map(batch, i, ref_res, what):
    mask = batch.mask_u8[i].cpu().numpy()
    thr = batch.thresholds[i].cpu().numpy()
    assert np.array_equal(mask, ref_res.mask), f"{what}: mask"
    assert np.array_equal(batch.mask(i), ref_res.mask), f"{what}: bit-packed mask"
    assert_bitwise(thr, ref_res.threshold_map, f"{what}: thresholds")
    d = batch.detections(i)
    r = ref_res.detections
    assert len(d) == len(r), f"{what}: {len(d)} vs {len(r)} detections"
    assert np.array_equal(d["row"], r["row"]) and np.array_equal(d["col"], r["col"]), f"{what}: order"
    assert_bitwise(d["value"], r["value"], f"{what}: values")
    assert_bitwise(d["threshold"], r["threshold"], f"{what}: det thresholds")


@pytest.mark.parametrize("fused", [False, True], ids=["two_kernel", "fused"])
def test_cfg3_maps_bit_identical_to_reference(uwb, ref, cuda, fused):
    """Config 3 maps (1024x1024 fp32, Exp(1) + 32 targets, g2 b8 pfa 1e-4), through
    SAT + ring CFAR (the default) and through the fused kernel (flags bit 4)."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    n = 6
    maps = synth.cfg3_maps(n, seed=3, device=cuda)
    p = uwb.CfarParams(2, 8, 1e-4)
    b = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=1024, want_mask_u8=True, want_thresholds=True)
    b(maps, fused=fused)
    torch.cuda.synchronize()
    b.check_inputs()
    host = maps.double().cpu().numpy()
    for i in range(n):
        _check_map(b, i, ref.cfar2d(host[i], 2, 8, 1e-4, "integral"), f"cfg3 map {i}")
    # mask bits only (the fast paths), compared with the reference masks
    b2 = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=1024)
    b2(maps, fused=fused)
    torch.cuda.synchronize()
    for i in range(n):
        assert np.array_equal(b2.mask(i), b.mask_u8[i].cpu().numpy()), f"cfg3 map {i} bits-only mask"
        assert b2.detections(i).tobytes() == b.detections(i).tobytes(), f"cfg3 map {i} bits-only detections"
    assert (b.detection_counts() >= 20).all()  # most of the 32 targets are found


def test_cfg1_map_and_sat(uwb, ref, cuda):
    """Config 1: one fp64 256x512 map, 5 targets at 15 dB, g2 b8 pfa 1e-4; output mask + SAT."""
    from paper_2012_11077_b200 import synth
    m = synth.cfg1_map(seed=1, device=cuda).cpu().numpy()
    got = uwb.cfar2d_integral(m, uwb.CfarParams(2, 8, 1e-4))
    exp = ref.cfar2d(m, 2, 8, 1e-4, "integral")
    assert np.array_equal(got.mask, exp.mask)
    assert_bitwise(got.threshold_map, exp.threshold_map, "cfg1 thresholds")
    assert_bitwise(uwb.build_sat(m).table(), ref.build_sat(m), "cfg1 SAT")
    assert len(got.detections) >= 5


@pytest.mark.parametrize("fused", [False, True], ids=["two_kernel", "fused"])
@pytest.mark.parametrize("win", [((1, 3), (4, 16)), ((3, 1), (16, 4))])
@pytest.mark.parametrize("pfa", [1e-3, 1e-5])
def test_cfg5_per_axis_windows_vs_restatement(uwb, oracle, cuda, win, pfa, fused):
    """Config 5 (K-clutter, non-square windows), scaled to 3 maps of 1024x512;
    per-cell outputs, then mask bits only (the fast paths)."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    (gr, gc), (br, bc) = win
    maps = synth.cfg5_maps(3, seed=5, device=cuda, rows=1024, cols=512)
    p = uwb.CfarParams(guard_radius=gr, background_radius=br, pfa=pfa, guard_cols=gc, background_cols=bc)
    b = BatchCfar(3, 1024, 512, p, torch.float32, det_capacity=4096, want_mask_u8=True, want_thresholds=True)
    b(maps, fused=fused)
    b2 = BatchCfar(3, 1024, 512, p, torch.float32, det_capacity=4096)
    b2(maps, fused=fused)
    torch.cuda.synchronize()
    host = maps.double().cpu().numpy()
    for i in range(3):
        exp = oracle.cfar(host[i], gr, gc, br, bc, pfa)
        _check_map(b, i, exp, f"cfg5 map {i}")
        assert np.array_equal(b2.mask(i), exp.mask), f"cfg5 map {i} bits-only mask"
        assert b2.detections(i).tobytes() == b.detections(i).tobytes(), f"cfg5 map {i} bits-only detections"


def test_slab_mode_vs_restatement_and_reference(uwb, ref, oracle, cuda):
    """Config 4 decomposition (row slabs, slab-local tables, global clamps) on a
    2048x1024 map with g4 b32 pfa 1e-5: bit-identical to the restatement with the
    same slabs; vs the reference's global table: masks equal outside a 1e-6 tie
    band and thresholds within 1e-9 relative."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    m = synth.cfg4_map(seed=4, device=cuda, rows=2048, cols=1024)
    p = uwb.CfarParams(4, 32, 1e-5)
    slab = 512
    b = BatchCfar(1, 2048, 1024, p, torch.float32, sat_mode="slab", slab_rows=slab, det_capacity=8192,
                  want_mask_u8=True, want_thresholds=True)
    b(m.unsqueeze(0).contiguous())
    torch.cuda.synchronize()
    host = m.double().cpu().numpy()
    thr = b.thresholds[0].cpu().numpy()
    mask = b.mask_u8[0].cpu().numpy()
    exp_thr = np.zeros_like(host)
    exp_mask = np.zeros(host.shape, np.uint8)
    for s0 in range(0, 2048, slab):
        r = oracle.cfar(host, 4, 4, 32, 32, 1e-5, row_begin=s0, row_end=s0 + slab, slab_local=True)
        exp_thr[s0:s0 + slab] = r.threshold_map[s0:s0 + slab]
        exp_mask[s0:s0 + slab] = r.mask[s0:s0 + slab]
    assert_bitwise(thr, exp_thr, "slab thresholds vs restatement")
    assert np.array_equal(mask, exp_mask)
    g = ref.cfar2d(host, 4, 32, 1e-5, "integral")
    rel = np.abs(thr - g.threshold_map) / np.maximum(g.threshold_map, 1e-300)
    assert rel.max() < 1e-9
    tie = np.abs(host - g.threshold_map) <= 1e-6 * g.threshold_map
    assert np.array_equal(mask[~tie], g.mask[~tie])


def test_wide_map_strip_chain_and_big_lists(uwb, ref, cuda):
    """Maps wider than one 1024-column strip chain their SAT strips; lists longer
    than one shared-memory sort run use the merge path."""
    from paper_2012_11077_b200.batch import BatchCfar
    g = torch.Generator(device="cuda").manual_seed(17)
    maps = torch.empty((2, 700, 3100), device="cuda", dtype=torch.float32).exponential_(1.0, generator=g)
    p = uwb.CfarParams(1, 3, 0.05)
    b = BatchCfar(2, 700, 3100, p, torch.float32, det_capacity=1 << 17, want_mask_u8=True,
                  want_thresholds=True)
    b(maps)
    torch.cuda.synchronize()
    host = maps.double().cpu().numpy()
    for i in range(2):
        _check_map(b, i, ref.cfar2d(host[i], 1, 3, 0.05, "integral"), f"wide map {i}")
    assert (b.detection_counts() > 2048).all()


def test_batch_reports_bad_cells(uwb, cuda):
    from paper_2012_11077_b200.batch import BatchCfar
    maps = torch.ones((3, 64, 64), device="cuda")
    maps[1, 5, 7] = float("nan")
    maps[2, 9, 1] = -1.0
    b = BatchCfar(3, 64, 64, uwb.CfarParams(1, 2, 1e-3), torch.float32)
    b(maps)
    torch.cuda.synchronize()
    fb = b.first_bad.cpu().numpy().astype(np.uint64)
    assert fb[1, 0] == 5 * 64 + 7 and fb[2, 1] == 9 * 64 + 1
    with pytest.raises(uwb.InputError) as e:
        b.check_inputs()
    assert str(e.value) == "build_sat: non-finite entry at (5, 7)"


def test_host_batch_e2e_matches_device_batch(uwb, cuda):
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar, host_cfar2d_batch
    n = 10
    maps = synth.cfg3_maps(n, seed=33, device=cuda)
    p = uwb.CfarParams(2, 8, 1e-4)
    b = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=512)
    b(maps)
    torch.cuda.synchronize()
    host_in = maps.cpu().pin_memory()
    bits = torch.zeros((n, 1024, 32), dtype=torch.int32).pin_memory()
    dets = torch.zeros((n, 512, 32), dtype=torch.uint8).pin_memory()
    counts = torch.zeros(n, dtype=torch.int64).pin_memory()
    host_cfar2d_batch(host_in, p, bits, dets, counts, 512, maps_per_chunk=3)
    assert torch.equal(bits, b.mask_bits.cpu())
    assert torch.equal(counts, b.counts.cpu())
    for i in range(n):
        k = int(counts[i])
        assert torch.equal(dets[i, :k], b.dets[i, :k].cpu())


@pytest.mark.parametrize("bad", ["nan", "inf", "neg", "nan_after_neg"])
def test_host_batch_rejects_bad_cells(uwb, cuda, bad):
    """uwb_host_cfar2d_batch raises what cfar2d_integral raises on the first bad
    map: build_sat's non-finite check (sat.cpp:28-32) before run_cfar's
    negative-power check (cfar.cpp:85-92), at the first row-major cell."""
    from paper_2012_11077_b200.batch import host_cfar2d_batch
    n, R, Cc = 5, 64, 96
    maps = torch.rand((n, R, Cc), dtype=torch.float32) + 0.1
    if bad == "nan":
        maps[3, 10, 11] = float("nan")
        maps[4, 1, 1] = float("nan")
        msg = "build_sat: non-finite entry at (10, 11)"
    elif bad == "inf":
        maps[2, 0, 95] = float("inf")
        msg = "build_sat: non-finite entry at (0, 95)"
    elif bad == "neg":
        maps[1, 63, 2] = -1.0
        maps[1, 63, 5] = -2.0
        msg = "cfar2d: cell (63, 2) is not a finite non-negative power"
    else:
        maps[2, 0, 0] = -1.0
        maps[2, 9, 9] = float("nan")
        msg = "build_sat: non-finite entry at (9, 9)"
    host_in = maps.pin_memory()
    bits = torch.zeros((n, R, 3), dtype=torch.int32).pin_memory()
    dets = torch.zeros((n, 64, 32), dtype=torch.uint8).pin_memory()
    counts = torch.zeros(n, dtype=torch.int64).pin_memory()
    with pytest.raises(uwb.InputError) as e:
        host_cfar2d_batch(host_in, uwb.CfarParams(1, 4, 1e-3), bits, dets, counts, 64, maps_per_chunk=2)
    assert str(e.value) == msg


@pytest.mark.parametrize("world", [2, 3])
def test_row_window_ranks_vs_restatement(uwb, oracle, cuda, world):
    """Config 4 sharded by rows: each "rank" holds only its owned rows
    plus the g+b halo (shard.row_slab) and runs uwb_dev_cfar2d_window with global
    row clamps. Ranks run one after another on this GPU; every slab is
    bit-identical to the restatement with the same row range and slab-local table,
    and detections carry global rows."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    from paper_2012_11077_b200.shard import row_slab
    rows, cols = 1500, 700
    m = synth.cfg4_map(seed=11, device=cuda, rows=rows, cols=cols)
    p = uwb.CfarParams(4, 32, 1e-5)
    host = m.double().cpu().numpy()
    halo = 4 + 32
    total = 0
    for rank in range(world):
        s = row_slab(rows, world, rank, halo)
        local = m[s.load_begin:s.load_end].contiguous().unsqueeze(0)
        b = BatchCfar(1, s.load_end - s.load_begin, cols, p, torch.float32, det_capacity=8192,
                      want_mask_u8=True, want_thresholds=True,
                      window=(rows, s.load_begin, s.owned_begin, s.owned_end))
        b(local)
        torch.cuda.synchronize()
        r = oracle.cfar(host, 4, 4, 32, 32, 1e-5, row_begin=s.owned_begin, row_end=s.owned_end, slab_local=True)
        own = slice(s.owned_begin, s.owned_end)
        assert_bitwise(b.thresholds[0].cpu().numpy(), r.threshold_map[own], f"rank {rank} thresholds")
        assert np.array_equal(b.mask_u8[0].cpu().numpy(), r.mask[own])
        assert np.array_equal(b.mask(0), r.mask[own])
        d = b.detections(0)
        exp = r.detections
        assert len(d) == len(exp)
        assert np.array_equal(d["row"], exp["row"]) and np.array_equal(d["col"], exp["col"])
        assert_bitwise(d["threshold"], exp["threshold"], "detection thresholds")
        total += len(d)
    assert total > 0


def test_row_window_rejects_missing_halo(uwb, cuda):
    from paper_2012_11077_b200.batch import BatchCfar
    from paper_2012_11077_b200.errors import BoundsError
    p = uwb.CfarParams(2, 8, 1e-4)
    local = torch.ones((1, 100, 64), device=cuda)
    # owned rows [200, 300) need rows [190, 310); the buffer starts at 200
    with pytest.raises(BoundsError):
        b = BatchCfar(1, 100, 64, p, torch.float32, window=(1000, 200, 200, 300))
        b(local)


def test_reused_tables_match_fresh_call(uwb, oracle, cuda):
    """flags bit 2: a second parameter set on the tables left in a shared
    workspace gives exactly the outputs of a fresh call."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    maps = synth.cfg5_maps(2, seed=9, device=cuda, rows=600, cols=500)
    pa = uwb.CfarParams(guard_radius=1, background_radius=4, pfa=1e-3, guard_cols=3, background_cols=16)
    pb = uwb.CfarParams(guard_radius=3, background_radius=16, pfa=1e-5, guard_cols=1, background_cols=4)
    a = BatchCfar(2, 600, 500, pa, torch.float32, det_capacity=8192, want_mask_u8=True, want_thresholds=True)
    b = BatchCfar(2, 600, 500, pb, torch.float32, det_capacity=8192, want_mask_u8=True, want_thresholds=True,
                  workspace=a.workspace)
    a(maps)
    b(maps, reuse_tables=True)
    torch.cuda.synchronize()
    host = maps.double().cpu().numpy()
    for i in range(2):
        _check_map(b, i, oracle.cfar(host[i], 3, 1, 16, 4, 1e-5), f"reused tables map {i}")
        _check_map(a, i, oracle.cfar(host[i], 1, 3, 4, 16, 1e-3), f"first call map {i}")


def test_naive_backend_flag_matches_reference_naive(uwb, ref, cuda):
    """flags bit 3 (naive backend, cfar.cpp:200-216) on the device batch path."""
    from paper_2012_11077_b200.batch import BatchCfar
    g = torch.Generator(device="cuda").manual_seed(23)
    maps = torch.empty((2, 96, 130), device="cuda", dtype=torch.float64).exponential_(1.0, generator=g)
    p = uwb.CfarParams(4, 8, 1e-3)
    b = BatchCfar(2, 96, 130, p, torch.float64, det_capacity=4096, want_mask_u8=True, want_thresholds=True)
    b(maps, naive=True)
    torch.cuda.synchronize()
    host = maps.cpu().numpy()
    for i in range(2):
        _check_map(b, i, ref.cfar2d(host[i], 4, 8, 1e-3, "naive"), f"naive map {i}")


@pytest.mark.parametrize("rows", [268, 270, 300, 33, 45, 262])
@pytest.mark.parametrize("fixed", [False, True], ids=["adaptive_chunks", "256_row_chunks"])
def test_ring_row_chunk_edges_bits_only(uwb, ref, cuda, rows, fixed):
    """The ring kernel's steady loop (taken only without per-cell outputs) on row
    counts whose last row chunk ends within the window of the bottom edge, with
    the adaptive (short) row chunks of small batches and with 256-row chunks
    (flags bit 8): masks and detection lists equal the reference."""
    from paper_2012_11077_b200.batch import BatchCfar
    gen = torch.Generator(device="cuda").manual_seed(rows)
    n, C = 3, 520
    maps = torch.empty((n, rows, C), device=cuda, dtype=torch.float32).exponential_(1.0, generator=gen)
    maps[:, ::9, ::7] *= 30.0
    p = uwb.CfarParams(2, 8, 1e-2)
    b = BatchCfar(n, rows, C, p, torch.float32, det_capacity=1 << 14)
    b(maps, exact=True, fixed_ring_rows=fixed)
    torch.cuda.synchronize()
    host = maps.double().cpu().numpy()
    for i in range(n):
        exp = ref.cfar2d(host[i], 2, 8, 1e-2, "integral")
        assert np.array_equal(b.mask(i), exp.mask), f"rows {rows} map {i}: mask"
        d = b.detections(i)
        assert np.array_equal(d["row"], exp.detections["row"]) and np.array_equal(d["col"], exp.detections["col"])
        assert_bitwise(d["threshold"], exp.detections["threshold"], f"rows {rows} map {i}: thresholds")


@pytest.mark.parametrize("rows,cols", [(256, 256), (512, 512)])
@pytest.mark.parametrize("certify", [False, True])
def test_long_lists_merge_passes_vs_reference(uwb, ref, cuda, rows, cols, certify):
    """Single maps (fewer lists than SMs: multi-CTA merge passes) with ~5k and
    ~21k detections in a 65536-entry list: the runs need 2 and 4 merge passes
    against the capacity's 5 (an odd / even pass count below the capacity's),
    and the sorted lists must equal the reference's (cfar.cpp:170-173)."""
    from paper_2012_11077_b200.batch import BatchCfar
    gen = torch.Generator(device="cuda").manual_seed(rows)
    maps = torch.empty((1, rows, cols), device=cuda, dtype=torch.float32).exponential_(1.0, generator=gen)
    p = uwb.CfarParams(1, 4, 0.08)  # (g + b, g) = (5, 1): a certified-path window
    b = BatchCfar(1, rows, cols, p, torch.float32, det_capacity=1 << 16)
    b(maps, certify=certify)
    torch.cuda.synchronize()
    n = int(b.counts[0])
    assert 4000 < n < 30000
    exp = ref.cfar2d(maps[0].double().cpu().numpy(), 1, 4, 0.08, "integral")
    d = b.detections(0)
    assert len(d) == len(exp.detections)
    assert np.array_equal(d["row"], exp.detections["row"]) and np.array_equal(d["col"], exp.detections["col"])
    assert_bitwise(d["value"], exp.detections["value"], "values")
    assert_bitwise(d["threshold"], exp.detections["threshold"], "thresholds")
