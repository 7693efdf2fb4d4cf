"""UWB_SAT_TILE (row slabs x column bands, one table per tile; the single-map
throughput mode of config 4) against the reference run on every tile's buffer.

Each owned cell's clamped window lies inside its tile's buffer and the buffer's
edges are map edges wherever the window clamps (paper_2012_11077_b200.shard.tiles),
so the tile CFAR must equal uwbvital_ref::cfar2d_integral (square windows) or the
C restatement (per-axis windows) run on the buffer alone: masks, thresholds and
detection lists bit-identical. Against the global table the masks agree outside
the 1e-6 tie band (north star)."""
import numpy as np
import pytest
import torch

from tests.helpers import assert_bitwise

pytestmark = pytest.mark.gpu


def _expected(host, tiles, run):
    thr = np.zeros_like(host)
    mask = np.zeros(host.shape, np.uint8)
    dets = []
    for t in tiles:
        (r0, r1), (c0, c1) = t.owned_rows, t.owned_cols
        (b0, b1), (d0, d1) = t.buf_rows, t.buf_cols
        res = run(np.ascontiguousarray(host[b0:b1, d0:d1]))
        thr[r0:r1, c0:c1] = res.threshold_map[r0 - b0:r1 - b0, c0 - d0:c1 - d0]
        mask[r0:r1, c0:c1] = res.mask[r0 - b0:r1 - b0, c0 - d0:c1 - d0]
        d = res.detections.copy()
        d["row"] += b0
        d["col"] += d0
        keep = (d["row"] >= r0) & (d["row"] < r1) & (d["col"] >= c0) & (d["col"] < c1)
        dets.append(d[keep])
    d = np.concatenate(dets)
    order = np.lexsort((d["col"], d["row"], -d["value"]))
    return mask, thr, d[order]


def _run_tiles(uwb, m, p, slab_rows, dtype, monkeypatch=None):
    from paper_2012_11077_b200.batch import BatchCfar
    rows, cols = m.shape
    b = BatchCfar(1, rows, cols, p, dtype, sat_mode="tile", slab_rows=slab_rows, det_capacity=1 << 16,
                  want_mask_u8=True, want_thresholds=True)
    b(m.unsqueeze(0).contiguous())
    torch.cuda.synchronize()
    b.check_inputs()
    return b


def _compare(b, mask, thr, dets, what):
    assert_bitwise(b.thresholds[0].cpu().numpy(), thr, f"{what}: thresholds")
    assert np.array_equal(b.mask_u8[0].cpu().numpy(), mask), f"{what}: mask"
    assert np.array_equal(b.mask(0), mask), f"{what}: bit-packed mask"
    d = b.detections(0)
    assert len(d) == len(dets), f"{what}: {len(d)} vs {len(dets)} detections"
    assert np.array_equal(d["row"], dets["row"]) and np.array_equal(d["col"], dets["col"]), f"{what}: order"
    assert_bitwise(d["value"], dets["value"], f"{what}: values")
    assert_bitwise(d["threshold"], dets["threshold"], f"{what}: det thresholds")


@pytest.mark.parametrize("rows,cols,slab", [(2048, 4096, 512), (1500, 2304, 0), (700, 3200, 256)])
def test_tiles_square_window_vs_reference_per_tile(uwb, ref, cuda, rows, cols, slab):
    """Config-4 window (g4 b32 pfa 1e-5, halo 64 columns) on maps cut into 4x4,
    2x3 (partial last band) and 3x4 tiles; plus the global table modulo the tie band."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.shard import tiles
    m = synth.cfg4_map(seed=7 + rows, device=cuda, rows=rows, cols=cols)
    p = uwb.CfarParams(4, 32, 1e-5)
    b = _run_tiles(uwb, m, p, slab, torch.float32)
    host = m.double().cpu().numpy()
    ts = tiles(rows, cols, 4, 4, 32, 32, slab)
    assert len({t.buf_cols for t in ts}) > 1
    mask, thr, dets = _expected(host, ts, lambda s: ref.cfar2d(s, 4, 32, 1e-5, "integral"))
    _compare(b, mask, thr, dets, f"tiles {rows}x{cols} slab {slab}")
    g = ref.cfar2d(host, 4, 32, 1e-5, "integral")
    tie = np.abs(host - g.threshold_map) <= 1e-6 * g.threshold_map
    assert np.array_equal(mask[~tie], g.mask[~tie])
    assert (np.abs(thr - g.threshold_map) / np.maximum(g.threshold_map, 1e-300)).max() < 1e-9


@pytest.mark.parametrize("win", [(1, 3, 4, 16), (3, 1, 16, 4)])
def test_tiles_per_axis_windows_vs_restatement(uwb, oracle, cuda, win):
    """Config-5 windows (column halo 32 / 32 after rounding; 1088-column band
    tables) on an 1100x2560 K-clutter map, fp64 input."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.shard import tiles
    gr, gc, br, bc = win
    m = synth.cfg5_maps(1, seed=11, device=cuda, rows=1100, cols=2560)[0].double()
    p = uwb.CfarParams(gr, br, 1e-3, guard_cols=gc, background_cols=bc)
    b = _run_tiles(uwb, m, p, 512, torch.float64)
    host = m.cpu().numpy()
    ts = tiles(1100, 2560, gr, gc, br, bc, 512)
    mask, thr, dets = _expected(host, ts, lambda s: oracle.cfar(s, gr, gc, br, bc, 1e-3))
    _compare(b, mask, thr, dets, f"per-axis {win}")


def test_tiles_unaligned_width_falls_back_to_row_slabs(uwb, oracle, cuda):
    """cols % 32 != 0: tile mode keeps row slabs only (the slab-mode result)."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    m = synth.cfg4_map(seed=3, device=cuda, rows=1024, cols=2500)
    p = uwb.CfarParams(2, 8, 1e-4)
    t = _run_tiles(uwb, m, p, 256, torch.float32)
    s = BatchCfar(1, 1024, 2500, p, torch.float32, sat_mode="slab", slab_rows=256, det_capacity=1 << 16,
                  want_mask_u8=True, want_thresholds=True)
    s(m.unsqueeze(0).contiguous())
    torch.cuda.synchronize()
    assert_bitwise(t.thresholds[0].cpu().numpy(), s.thresholds[0].cpu().numpy(), "thresholds")
    assert t.detections(0).tobytes() == s.detections(0).tobytes()


def test_tiles_report_first_bad_cell_in_map_coordinates(uwb, cuda):
    """A non-finite cell inside a band's halo is reported at its map (row, col)."""
    from paper_2012_11077_b200.batch import BatchCfar
    from paper_2012_11077_b200.errors import InputError
    m = torch.rand(600, 4096, device=cuda, dtype=torch.float32)
    m[300, 2050] = float("nan")
    m[450, 1000] = float("inf")
    b = BatchCfar(1, 600, 4096, uwb.CfarParams(4, 32, 1e-5), torch.float32, sat_mode="tile", slab_rows=256)
    b(m.unsqueeze(0))
    torch.cuda.synchronize()
    with pytest.raises(InputError) as e:
        b.check_inputs()
    assert "(300, 2050)" in str(e.value)


@pytest.mark.parametrize("world", [2, 3])
def test_row_window_col_bands_ranks_vs_reference_per_tile(uwb, ref, cuda, world):
    """Config-4 sharding with column bands (bench.py --config 4 at any N): each
    rank holds its row slab + halo and runs uwb_dev_cfar2d_window with col_bands;
    every tile equals the reference run on the tile's buffer."""
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    from paper_2012_11077_b200.shard import row_slab, tiles
    rows, cols, halo = 1800, 3072, 36
    m = synth.cfg4_map(seed=21, device=cuda, rows=rows, cols=cols)
    host = m.double().cpu().numpy()
    p = uwb.CfarParams(4, 32, 1e-5)
    per = -(-rows // world)
    mask, thr, dets = _expected(host, tiles(rows, cols, 4, 4, 32, 32, per, 1024),
                                lambda s: ref.cfar2d(s, 4, 32, 1e-5, "integral"))
    got = []
    for rank in range(world):
        s = row_slab(rows, world, rank, halo)
        local = m[s.load_begin:s.load_end].contiguous().unsqueeze(0)
        b = BatchCfar(1, s.load_end - s.load_begin, cols, p, torch.float32, det_capacity=1 << 15,
                      want_mask_u8=True, want_thresholds=True,
                      window=(rows, s.load_begin, s.owned_begin, s.owned_end, 1024))
        b(local)
        torch.cuda.synchronize()
        o0, o1 = s.owned_begin, s.owned_end
        assert_bitwise(b.thresholds[0].cpu().numpy(), thr[o0:o1], f"rank {rank} thresholds")
        assert np.array_equal(b.mask(0), mask[o0:o1]), f"rank {rank} mask"
        got.append(b.detections(0))
    d = np.concatenate(got)
    d = d[np.lexsort((d["col"], d["row"], -d["value"]))]
    assert d.tobytes() == dets.tobytes()
