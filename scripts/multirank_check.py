"""Rank program of the multi-rank checks (tests/test_gpu_multirank.py).

Launched under torch.distributed.run with 1 or N ranks. Every rank runs the
product path on its shard exactly as bench.py / bench_configs.py do:

* batched maps (config 3 shape): bench._shard -> bench._generate -> BatchCfar
  -> detection-count all-reduce (shard.reduce_count);
* one large map (config 4 decomposition, smaller): shard.row_slab -> the rank
  loads its owned rows plus the g+b halo -> uwb_dev_cfar2d_window with global
  row clamps and 1024-column tile tables -> count all-reduce.

Each rank writes its per-map counts, mask bits, detection lists and the reduced
totals to ``--out``/rank<k>.npz; the test concatenates them and compares the
world-N run with the world-1 run (bit-identical: the same kernels run on the
same maps / tiles). UWB_DIST_BACKEND=gloo lets N ranks share one GPU (no kernel
of one rank waits on another rank; the count reduce goes through gloo).
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--maps", type=int, default=256)
    ap.add_argument("--big-rows", type=int, default=4096)
    ap.add_argument("--big-cols", type=int, default=4096)
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    import bench as B
    import paper_2012_11077_b200 as uwb
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    from paper_2012_11077_b200.shard import reduce_count, row_slab

    world, rank, local = B._dist()
    dev = B._init_rank(world, local)
    B.N_MAPS = args.maps

    # ---- batched maps: bench.py's shard / generator / count reduce ----
    m0, m1 = B._shard(world, rank)
    maps = B._generate(m0, m1, dev)
    p3 = uwb.CfarParams(B.GUARD, B.TRAIN, B.PFA)
    runner = BatchCfar(m1 - m0, B.ROWS, B.COLS, p3, torch.float32, det_capacity=512, device=dev)
    runner(maps)
    total = runner.counts.sum().view(1).clone()
    reduce_count(total)
    torch.cuda.synchronize()
    runner.check_inputs()
    dets = [runner.detections(i) for i in range(m1 - m0)]

    # ---- one large map in row slabs with a g+b halo ----
    R, C = args.big_rows, args.big_cols
    g, b, pfa = 4, 32, 1e-5
    s = row_slab(R, world, rank, g + b)
    full = synth.cfg4_map(seed=4, device=dev, rows=R, cols=C)
    slab = full[s.load_begin:s.load_end].contiguous().unsqueeze(0)
    del full
    big = BatchCfar(1, s.load_end - s.load_begin, C, uwb.CfarParams(g, b, pfa), torch.float32,
                    det_capacity=1 << 14, slab_rows=512, device=dev,
                    window=(R, s.load_begin, s.owned_begin, s.owned_end, 1024))
    big(slab)
    big_total = big.counts.sum().view(1).clone()
    reduce_count(big_total)
    torch.cuda.synchronize()
    big_dets = big.detections(0)

    os.makedirs(args.out, exist_ok=True)
    np.savez(os.path.join(args.out, f"rank{rank}.npz"),
             world=world, m0=m0, m1=m1,
             counts=runner.counts.cpu().numpy(), mask_bits=runner.mask_bits.cpu().numpy(),
             dets=np.concatenate(dets) if dets else np.zeros(0, dtype=uwb.DETECTION_DTYPE),
             total=int(total.item()),
             owned=(s.owned_begin, s.owned_end), big_mask_bits=big.mask_bits[0].cpu().numpy(),
             big_dets=big_dets, big_total=int(big_total.item()), big_count=int(big.counts[0].item()))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
