"""Host-side checks of the UWB_SAT_TILE decomposition (shard.tiles): owned cells
covered exactly once, uniform 32-aligned band tables inside the map, and every
owned cell's window inside its buffer with the buffer edge a map edge wherever the
window clamps (the property that makes a tile's CFAR the reference's CFAR of the
buffer)."""
import numpy as np
import pytest

from paper_2012_11077_b200.shard import tiles


@pytest.mark.parametrize("rows,cols,g,b,slab,band", [
    (16384, 16384, (4, 4), (32, 32), 0, 1024), (2048, 4096, (4, 4), (32, 32), 512, 1024),
    (1500, 2304, (4, 4), (32, 32), 0, 1024), (1100, 2560, (1, 3), (4, 16), 512, 1024),
    (1100, 2560, (3, 1), (16, 4), 512, 1000), (700, 2500, (2, 2), (8, 8), 256, 1024),
    (300, 1024, (2, 2), (8, 8), 0, 1024)])
def test_tile_cover_and_windows(rows, cols, g, b, slab, band):
    ts = tiles(rows, cols, g[0], g[1], b[0], b[1], slab, band)
    cover = np.zeros((rows, cols), np.int32)
    widths = set()
    hr, hc = g[0] + b[0], g[1] + b[1]
    for t in ts:
        (r0, r1), (c0, c1) = t.owned_rows, t.owned_cols
        (b0, b1), (d0, d1) = t.buf_rows, t.buf_cols
        cover[r0:r1, c0:c1] += 1
        widths.add(d1 - d0)
        assert 0 <= b0 <= r0 < r1 <= b1 <= rows and 0 <= d0 <= c0 < c1 <= d1 <= cols
        assert d0 % 32 == 0
        # clamped windows of the owned corners lie in the buffer ...
        assert max(0, r0 - hr) >= b0 and min(rows, r1 - 1 + hr + 1) <= b1
        assert max(0, c0 - hc) >= d0 and min(cols, c1 - 1 + hc + 1) <= d1
        # ... and where the buffer edge is not a map edge no owned window reaches it
        assert b0 == 0 or r0 - hr >= b0
        assert d0 == 0 or c0 - hc >= d0
        assert b1 == rows or r1 - 1 + hr < b1
        assert d1 == cols or c1 - 1 + hc < d1
    assert (cover == 1).all()
    assert len(widths) == 1
