"""Multi-GPU partitioning of the north-star path.

* Batched maps (configs 3 and 5): maps are independent units; each rank owns a
  contiguous block of whole maps (in blocks of ``block`` maps so the seeded
  generator produces the same bytes whatever the world size). No data-path
  collective; the only exchange is the per-batch detection-count all-reduce.
* One large map (config 4): rank g owns rows [r0, r1) and loads the halo rows
  [l0, l1) = [r0 - h, r1 + h) clipped to the map (h = g_r + b_r), builds a
  slab-local summed-area table and clamps windows with global row indices, so no
  cross-GPU prefix or halo exchange is needed at run time.
"""
from __future__ import annotations

from dataclasses import dataclass


def map_shard(n_maps: int, world: int, rank: int, block: int = 64) -> tuple[int, int]:
    """[m0, m1) of whole maps owned by `rank` (blocks of `block` maps; the
    remainder block, if any, goes to the last rank)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    blocks = (n_maps + block - 1) // block
    per, extra = divmod(blocks, world)
    b0 = rank * per + min(rank, extra)
    b1 = b0 + per + (1 if rank < extra else 0)
    return min(n_maps, b0 * block), min(n_maps, b1 * block)


@dataclass(frozen=True)
class RowSlab:
    owned_begin: int
    owned_end: int
    load_begin: int
    load_end: int

    @property
    def halo_above(self) -> int:
        return self.owned_begin - self.load_begin

    @property
    def halo_below(self) -> int:
        return self.load_end - self.owned_end


def row_slab(rows: int, world: int, rank: int, halo: int) -> RowSlab:
    """Rank's owned rows (ceil(rows/world) per rank) and the rows it must load."""
    per = (rows + world - 1) // world
    r0 = min(rows, rank * per)
    r1 = min(rows, r0 + per)
    return RowSlab(r0, r1, max(0, r0 - halo), min(rows, r1 + halo))


def reduce_count(count, group=None):
    """Sum a per-rank detection count tensor across ranks (NCCL on GPU, gloo on CPU)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(count, op=dist.ReduceOp.SUM, group=group)
    return count


@dataclass(frozen=True)
class Tile:
    """One table of UWB_SAT_TILE: owned rows/cols and the buffer its table covers."""
    owned_rows: tuple[int, int]
    owned_cols: tuple[int, int]
    buf_rows: tuple[int, int]
    buf_cols: tuple[int, int]


def tiles(rows: int, cols: int, guard_rows: int, guard_cols: int, background_rows: int,
          background_cols: int, slab_rows: int = 0, band_cols: int = 1024) -> list[Tile]:
    """Host mirror of the UWB_SAT_TILE decomposition (csrc/capi.cu make_plan,
    csrc/kernels.cuh JobGeometry::band_c0): row slabs of ``slab_rows`` (0 = 1024)
    owned rows with a g_r + b_r halo, column bands of ``band_cols`` (rounded up
    to 128) owned columns whose tables span band_cols + 2 hp source columns,
    hp = g_c + b_c rounded up to 32, moved inward at the map edges. Every owned
    cell's clamped window lies inside its tile's buffer and the buffer's edges
    are map edges wherever the window clamps, so the CFAR of a tile equals the
    reference's cfar2d_integral run on the buffer alone (the parity oracle)."""
    slab = slab_rows or 1024
    if slab >= rows:
        slab = rows
    hr = guard_rows + background_rows
    bc = -(-max(band_cols, 128) // 128) * 128
    hp = -(-(guard_cols + background_cols) // 32) * 32
    banded = cols % 32 == 0 and bc + 2 * hp < cols
    out = []
    for r0 in range(0, rows, slab):
        r1 = min(rows, r0 + slab)
        br = (max(0, r0 - hr), min(rows, r1 + hr)) if slab < rows else (0, rows)
        if not banded:
            out.append(Tile((r0, r1), (0, cols), br, (0, cols)))
            continue
        width = bc + 2 * hp
        for k in range(-(-cols // bc)):
            c0 = min(max(k * bc - hp, 0), cols - width)
            out.append(Tile((r0, r1), (k * bc, min(cols, (k + 1) * bc)), br, (c0, c0 + width)))
    return out
