"""CPU (gloo, world_size 2) coverage of the multi-GPU host logic: map sharding,
row-slab decomposition with halos, and the detection-count reduce. The CFAR of
each shard is computed here by the oracle restatement (slab-local tables), so
the test checks that the decomposition reproduces the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2012_11077_b200.shard import map_shard, reduce_count, row_slab


def test_map_shard_covers_every_map_once():
    for n_maps in (4096, 64, 130, 1):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                m0, m1 = map_shard(n_maps, world, r)
                seen.extend(range(m0, m1))
            assert seen == list(range(n_maps))


def test_row_slabs_cover_rows_with_halo():
    for rows, world, halo in [(16384, 8, 36), (100, 3, 5), (7, 4, 2)]:
        owned = []
        for r in range(world):
            s = row_slab(rows, world, r, halo)
            owned.extend(range(s.owned_begin, s.owned_end))
            assert s.load_begin == max(0, s.owned_begin - halo)
            assert s.load_end == min(rows, s.owned_end + halo)
        assert owned == list(range(rows))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import OracleLib
        o = OracleLib()
        rng = np.random.default_rng(99)
        big = rng.exponential(1.0, (96, 80))
        big[40, 20] += 60.0
        gr, br = 2, 6
        s = row_slab(96, world, rank, gr + br)
        # the rank only holds its loaded rows; windows clamp to the global map
        local = np.zeros_like(big)
        local[s.load_begin:s.load_end] = big[s.load_begin:s.load_end]
        res = o.cfar(local, gr, gr, br, br, 1e-3, row_begin=s.owned_begin, row_end=s.owned_end,
                     slab_local=True)
        count = torch.tensor([len(res.detections)], dtype=torch.int64)
        reduce_count(count)
        maps = list(range(*map_shard(256, world, rank)))
        n = torch.tensor([len(maps)], dtype=torch.int64)
        reduce_count(n)
        result_q.put((rank, int(count.item()), int(n.item()),
                      res.threshold_map[s.owned_begin:s.owned_end].copy(),
                      res.mask[s.owned_begin:s.owned_end].copy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_slab_decomposition_and_count_reduce():
    from oracle.pyoracle import OracleLib
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    rng = np.random.default_rng(99)
    big = rng.exponential(1.0, (96, 80))
    big[40, 20] += 60.0
    o = OracleLib()
    single = o.cfar(big, 2, 2, 6, 6, 1e-3)
    thr = np.concatenate([x[3] for x in out])
    mask = np.concatenate([x[4] for x in out])
    # slab-local tables re-associate the sums: thresholds agree to rounding,
    # masks agree outside the tie band
    assert np.max(np.abs(thr - single.threshold_map) / np.maximum(single.threshold_map, 1e-300)) < 1e-12
    tie = np.abs(big - single.threshold_map) <= 1e-9 * single.threshold_map
    assert np.array_equal(mask[~tie], single.mask[~tie])
    total = out[0][1]
    assert all(x[1] == total for x in out)
    assert total == int(mask.sum())
    assert all(x[2] == 256 for x in out)
