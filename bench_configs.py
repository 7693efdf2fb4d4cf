"""bench.py --config {1,2,4,5}: the other BASELINE.json workloads.

bench.py's default line is config 3 (the throughput config BASELINE's metric is
quoted on). These lines measure the remaining configurations with the same
JSON schema so every row of SURVEY 8d has a number:

* config 4 - one 16384 x 16384 fp32 map, g4 b32 Pfa 1e-5. One rank per GPU owns
  a row slab (shard.row_slab) and holds only its rows plus the g+b halo; the
  device path is uwb_dev_cfar2d_window (slab-local table, global clamps), then
  the detection-count all-reduce. value = whole-map cells / device time (max
  over ranks). At N=1 the window is the whole map, i.e. the reference-exact
  global table.
* config 5 - 64 K-clutter fp32 maps 8192 x 2048, the four runs (g_r,g_c,b_r,b_c)
  in {(1,3,4,16), (3,1,16,4)} x Pfa in {1e-3, 1e-5}; one step = all four runs;
  maps sharded across ranks. The reference cannot express per-axis windows, so
  its CPU baseline is the C restatement (kind "port").
* config 1 - one 256 x 512 fp64 map (launch-bound; ms_per_step is per map).
* config 2 - front end + CFAR of 512 x 1024 records, batched on the device
  (uwb_dev_detect_batch; value in records/s) with the host-level detect()
  latency of one record beside it.
* --config 6 - the paper's Table I: naive vs integral-image CA-CFAR on a
  1024 x 600 map for (g, b) in {(4,8), (4,12), (8,8), (8,12)}, GPU and reference.
"""
from __future__ import annotations

import json
import statistics
import time

import numpy as np

import bench as B


def _line(**kw):
    base = {"n_gpus": 1, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE generator)"}
    base.update(kw)
    print(json.dumps(base), flush=True)


def _events_time(fn, steps, warmup, world, dist):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item())


def _phases(n):
    """Mean {certify, sat, cfar, sort} ms of the last n phase-timed calls."""
    from paper_2012_11077_b200.batch import phase_ms4
    ph = phase_ms4(1024)[-n:]
    return {k: float(np.mean(ph[:, i])) for i, k in enumerate(("certify", "sat", "cfar", "sort"))} if len(ph) else {}


def _roof(phases, cells, peak, peak_src, certified=True):
    """Roofline of the dominant kernel (bench.step_kernels), plus the whole
    step's HBM fraction over the algorithmic bytes of all its kernels."""
    ks = B.step_kernels(phases.get("certify", 0.0), phases.get("sat", 0.0), phases.get("cfar", 0.0), cells,
                        certified)
    r = B.roofline_of(ks, peak, peak_src)
    r["bytes_per_cell"] = r["launch_bytes"] / cells
    return r


def _step_frac(phases, cells, ms, peak, certified=True):
    """Whole-step HBM fraction over the algorithmic bytes of the step's kernels."""
    ks = B.step_kernels(phases.get("certify", 0.0), phases.get("sat", 0.0), phases.get("cfar", 0.0), cells,
                        certified)
    return sum(v[1] for v in ks.values()) / (ms / 1e3) / 1e9 / peak


def _certified(runner) -> bool:
    return bool((runner.cert_status.cpu().numpy() == 0).all())


def _init_dist():
    import torch
    import torch.distributed as dist
    world, rank, local = B._dist()
    B._init_rank(world, local)
    return world, rank, dist


# ------------------------------------------------------------------ config 4 --
CFG4_SLAB_ROWS, CFG4_BAND_COLS = 512, 1024


def run_cfg4(args):
    import torch
    import paper_2012_11077_b200 as uwb
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar, kernel_launches
    from paper_2012_11077_b200.shard import reduce_count, row_slab
    world, rank, dist = _init_dist()
    R = C = 16384
    g, b, pfa = 4, 32, 1e-5
    s = row_slab(R, world, rank, g + b)
    full = synth.cfg4_map(seed=4, device="cuda", rows=R, cols=C)
    local = full[s.load_begin:s.load_end].contiguous().unsqueeze(0)
    host_full = full.cpu() if (rank == 0 and world == 1 and not args.no_cpu_baseline) else None
    del full
    p = uwb.CfarParams(g, b, pfa)
    # tiles: 512-row slabs x 1024-column bands inside the rank's row window, one
    # table per tile (UWB_SAT_TILE semantics): the map runs as a batch of short
    # SAT strip chains instead of one 128-strip chain (DESIGN 4(c))
    runner = BatchCfar(1, s.load_end - s.load_begin, C, p, torch.float32, det_capacity=1 << 16,
                       slab_rows=CFG4_SLAB_ROWS, tie_capacity=1 << 12,
                       window=(R, s.load_begin, s.owned_begin, s.owned_end, CFG4_BAND_COLS))
    count = torch.zeros(1, dtype=torch.int64, device="cuda")

    def step(phase=False):
        runner(local, phase_events=phase)
        count.copy_(runner.counts.sum().view(1))
        reduce_count(count)

    step(phase=True)
    from paper_2012_11077_b200.batch import phase_ms4
    phase_ms4(1024)
    sampler = B.ClockSampler(torch.cuda.current_device())
    sampler.start()
    l0 = kernel_launches()
    ms = _events_time(lambda: step(phase=True), args.steps, max(args.warmup - 1, 0), world, dist)
    launches = kernel_launches() - l0
    clocks = sampler.stop()
    ph = _phases(args.steps + max(args.warmup - 1, 0))
    owned_cells = (s.owned_end - s.owned_begin) * C
    peak, src = B._peaks()

    # end to end: pinned host slab -> H2D -> SAT+CFAR+sort -> D2H of mask and counts
    host = torch.empty(local.shape, dtype=torch.float32, pin_memory=True)
    host.copy_(local)
    dev_in = torch.empty_like(local)
    mask_host = torch.empty(runner.mask_bits.shape, dtype=torch.int32, pin_memory=True)
    cnt_host = torch.empty(1, dtype=torch.int64, pin_memory=True)

    def e2e_step():
        dev_in.copy_(host, non_blocking=True)
        runner(dev_in)
        mask_host.copy_(runner.mask_bits, non_blocking=True)
        cnt_host.copy_(runner.counts, non_blocking=True)
        torch.cuda.synchronize()

    e2e_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_step()
    e_ms = torch.tensor([(time.perf_counter() - t0) * 1e3 / args.e2e_steps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e_ms = float(e_ms.item())

    exact = None
    tie_check = {"tie_band_cells_tile": int(runner.tie_counts[0].item()), "tie_band": "|cut - T| <= 1e-6 T"}
    if world == 1:
        # the reference-exact global table (one 128-strip SAT chain) on the same map
        g_runner = BatchCfar(1, R, C, p, torch.float32, det_capacity=1 << 16, tie_capacity=1 << 12)
        g_count = torch.zeros(1, dtype=torch.int64, device="cuda")

        def g_step(phase=False):
            g_runner(local, phase_events=phase)
            g_count.copy_(g_runner.counts.sum().view(1))

        g_step()
        g_ms = _events_time(lambda: g_step(phase=True), max(3, args.steps // 2), 1, world, dist)
        g_ph = _phases(max(3, args.steps // 2) + 1)
        exact = {"value": R * C / (g_ms / 1e3) / 1e9, "unit": B.UNIT, "ms_per_step": g_ms, "phases_ms": g_ph,
                 "sat": "one global table (bit-identical to the reference)", "detections": int(g_count.item()),
                 "certified": _certified(g_runner)}
        # the tile path against the reference-exact global table on this map:
        # cells whose decision differs must all lie in the tie band
        runner(local)
        torch.cuda.synchronize()
        tb, gb = runner.mask_bits[0].cpu().numpy().view(np.uint32), g_runner.mask_bits[0].cpu().numpy().view(np.uint32)
        diff = np.argwhere(np.unpackbits((tb ^ gb).view(np.uint8), axis=1, bitorder="little")[:, :C])
        t_ties, g_ties = runner.tie_band(0), g_runner.tie_band(0)
        band = set(zip(t_ties["row"].tolist(), t_ties["col"].tolist())) | \
            set(zip(g_ties["row"].tolist(), g_ties["col"].tolist()))
        tie_check = {"tile_vs_global_differing_cells": int(len(diff)),
                     "differing_outside_tie_band": int(sum(1 for x in diff.tolist() if tuple(x) not in band)),
                     "tie_band_cells_tile": int(len(t_ties)), "tie_band_cells_global": int(len(g_ties)),
                     "tie_band": "|cut - T| <= 1e-6 T"}
        del g_runner

    cpu = None
    if host_full is not None:
        from oracle.pyoracle import RefLib
        cores = B._cpu_threads()
        secs, _ = RefLib().time_cfar_batch(host_full.numpy()[None], g, b, pfa, 1, ref_threads=cores)
        cpu = {"value": R * C / secs / 1e9, "unit": B.UNIT, "cores": cores, "kind": "reference",
               "sample": f"the whole config-4 map, uwbvital_ref::cfar2d_integral(map, params, {cores}) "
                         f"(the reference's own row threads; build_sat is serial), {secs:.2f} s"}
    if rank == 0:
        _line(metric=B.METRIC, value=R * C / (ms / 1e3) / 1e9, unit=B.UNIT, n_gpus=world, steps=args.steps,
              warmup=args.warmup, ms_per_step=ms,
              config={"workload": "cfg4: one 16384x16384 fp32 map, Exp(1) + 1000 3x3 targets at U(6,18) dB, "
                                  "guard 4, train 32, Pfa 1e-5",
                      "parallelism": f"row slabs over {world} GPU(s), halo {g + b} rows, global clamps "
                                     "(uwb_dev_cfar2d_window)",
                      "sat": f"tile-local tables ({CFG4_SLAB_ROWS}-row slabs x {CFG4_BAND_COLS}-column bands, "
                             "halo 36 rows / 64 columns): bit-identical to the reference run on each tile's "
                             "buffer; against the global table see tie_check (measured in this run at N=1)",
                      "l2": "1 GiB input + 2.1 GiB table per pass >> 126 MB L2",
                      "detections_per_step": int(count.item())},
              roofline=_roof(ph, owned_cells, peak, src, _certified(runner)), phases_ms=ph,
              step_hbm_frac=_step_frac(ph, owned_cells, ms, peak, _certified(runner)),
              global_exact=exact, tie_check=tie_check, cpu_baseline=cpu,
              e2e={"value": R * C / (e_ms / 1e3) / 1e9, "unit": B.UNIT,
                   "h2d_bytes_per_step": int(host.numel() * 4) * world,
                   "d2h_bytes_per_step": int(mask_host.numel() * 4 + 8) * world, "ms_per_step": e_ms,
                   "timer": "host wall clock, H2D + compute + D2H, max over ranks"},
              gpu_launches=int(launches), clocks=clocks)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------ config 5 --
CFG5_RUNS = [((1, 3, 4, 16), 1e-3), ((1, 3, 4, 16), 1e-5), ((3, 1, 16, 4), 1e-3), ((3, 1, 16, 4), 1e-5)]


def run_cfg5(args):
    import torch
    import paper_2012_11077_b200 as uwb
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar, host_cfar2d_batch, kernel_launches
    from paper_2012_11077_b200.shard import map_shard, reduce_count
    world, rank, dist = _init_dist()
    n_all, R, C = 64, 8192, 2048
    m0, m1 = map_shard(n_all, world, rank, block=8)
    maps = torch.empty((m1 - m0, R, C), dtype=torch.float32, device="cuda")
    for blk in range(m0 // 8, m1 // 8):
        maps[blk * 8 - m0:(blk + 1) * 8 - m0] = synth.cfg5_maps(8, seed=5_000 + blk, device="cuda", rows=R, cols=C)
    # the four runs share one workspace and run one after another; each is a
    # certified-path call (its own window-sum pass, sparse SAT and resolve:
    # 8 B/cell per run, against 12 + 4 x 12.125 B/cell for one full table read
    # back by the four parameter sets)
    runners = []
    for (gr, gc, br, bc), pfa in CFG5_RUNS:
        p = uwb.CfarParams(guard_radius=gr, background_radius=br, pfa=pfa, guard_cols=gc, background_cols=bc)
        runners.append(BatchCfar(m1 - m0, R, C, p, torch.float32, det_capacity=1 << 15,
                                 workspace=runners[0].workspace if runners else None))
    count = torch.zeros(1, dtype=torch.int64, device="cuda")

    def step(phase=False):
        count.zero_()
        for i, rn in enumerate(runners):
            rn(maps, phase_events=phase)
            count.add_(rn.counts.sum())
        reduce_count(count)

    step(phase=True)
    from paper_2012_11077_b200.batch import phase_ms4
    phase_ms4(1024)
    sampler = B.ClockSampler(torch.cuda.current_device())
    sampler.start()
    l0 = kernel_launches()
    ms = _events_time(lambda: step(phase=True), args.steps, max(args.warmup - 1, 0), world, dist)
    launches = kernel_launches() - l0
    clocks = sampler.stop()
    ph = _phases(4 * (args.steps + max(args.warmup - 1, 0)))  # per run (call)
    certified = all(_certified(rn) for rn in runners)
    cells_local = (m1 - m0) * R * C
    peak, src = B._peaks()

    # end to end through the host API, all four runs
    host = torch.empty(maps.shape, dtype=torch.float32, pin_memory=True)
    host.copy_(maps)
    outs = [(torch.empty(rn.mask_bits.shape, dtype=torch.int32, pin_memory=True),
             torch.empty((m1 - m0, rn.det_capacity, 32), dtype=torch.uint8, pin_memory=True),
             torch.empty(m1 - m0, dtype=torch.int64, pin_memory=True)) for rn in runners]

    def e2e_step():
        for rn, (bits, dets, cnt) in zip(runners, outs):
            host_cfar2d_batch(host, rn.params, bits, dets, cnt, rn.det_capacity, maps_per_chunk=4)

    e2e_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_step()
    e_ms = torch.tensor([(time.perf_counter() - t0) * 1e3 / args.e2e_steps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e_ms = float(e_ms.item())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle.pyoracle import OracleLib
        o = OracleLib()
        one = maps[0].double().cpu().numpy()
        t0 = time.perf_counter()
        for (gr, gc, br, bc), pfa in CFG5_RUNS:
            o.cfar(one, gr, gc, br, bc, pfa)
        secs = time.perf_counter() - t0
        cpu = {"value": 4 * R * C / secs / 1e9, "unit": B.UNIT, "cores": 1, "kind": "port",
               "sample": f"one config-5 map x the 4 runs through the C restatement (uwbo_cfar, 1 thread; the "
                         f"reference has no per-axis windows), {secs:.2f} s"}
    if rank == 0:
        total_cells = 4 * n_all * R * C
        _line(metric=B.METRIC, value=total_cells / (ms / 1e3) / 1e9, unit=B.UNIT, n_gpus=world, steps=args.steps,
              warmup=args.warmup, ms_per_step=ms,
              config={"workload": "cfg5: 64 K-clutter fp32 maps 8192x2048 (Gamma(0.5) texture, 16x16 box, "
                                  "x Exp(1) speckle) + 64 clusters/map at U(10,25) dB; windows (g_r,g_c,b_r,b_c) "
                                  "(1,3,4,16),(3,1,16,4) x Pfa 1e-3,1e-5; one step = the 4 runs, each a full "
                                  "certified-path call (the e2e leg runs the same 4 calls from host buffers)",
                      "parallelism": f"dp{world} (maps sharded in 8-map blocks)",
                      "l2": "4 GiB input per run >> 126 MB L2", "detections_per_step": int(count.item())},
              roofline=_roof(ph, cells_local, peak, src, certified), phases_ms_per_run=ph,
              step_hbm_frac=_step_frac(ph, cells_local, ms / 4, peak, certified), cpu_baseline=cpu,
              e2e={"value": total_cells / (e_ms / 1e3) / 1e9, "unit": B.UNIT,
                   "h2d_bytes_per_step": int(4 * host.numel() * 4) * world,
                   "d2h_bytes_per_step": int(sum(o[0].numel() * 4 + o[1].numel() + o[2].numel() * 8
                                                 for o in outs)) * world,
                   "ms_per_step": e_ms, "timer": "host wall clock around the synchronous calls"},
              gpu_launches=int(launches), clocks=clocks)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------ config 1 --
def run_cfg1(args):
    import torch
    import paper_2012_11077_b200 as uwb
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar, kernel_launches
    world, rank, dist = _init_dist()
    m = synth.cfg1_map(seed=1, device="cuda").unsqueeze(0).contiguous()
    p = uwb.CfarParams(2, 8, 1e-4)
    runner = BatchCfar(1, 256, 512, p, torch.float64, det_capacity=4096)
    l0 = kernel_launches()
    ms = _events_time(lambda: runner(m), args.steps, args.warmup, world, dist)
    launches = (kernel_launches() - l0) * args.steps // (args.steps + args.warmup)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        from oracle.pyoracle import RefLib
        ref = RefLib()
        host = m[0].cpu().numpy()
        ref.cfar2d(host, 2, 8, 1e-4)
        t0 = time.perf_counter()
        reps = 20
        for _ in range(reps):
            ref.cfar2d(host, 2, 8, 1e-4)
        secs = (time.perf_counter() - t0) / reps
        cpu = {"value": 256 * 512 / secs / 1e9, "unit": B.UNIT, "cores": 1, "kind": "reference",
               "sample": f"the config-1 map, uwbvital_ref::cfar2d_integral(map, params, 1) incl. threshold map, "
                         f"{secs * 1e3:.2f} ms"}
    if rank == 0:
        _line(metric=B.METRIC, value=256 * 512 / (ms / 1e3) / 1e9, unit=B.UNIT, n_gpus=world, steps=args.steps,
              warmup=args.warmup, ms_per_step=ms,
              config={"workload": "cfg1: one fp64 map 256x512, Exp(1) + 5 targets at 15 dB, guard 2, train 8, "
                                  "Pfa 1e-4 (launch-bound; ms_per_step is per map)", "parallelism": "replicas"},
              roofline=None, cpu_baseline=cpu, e2e=None, gpu_launches=int(launches), clocks=None)
    return 0


# ------------------------------------------------------------------ config 2 --
# Algorithmic fp64 operations per config-2 record (M = 512 fast-time samples x
# N = 1024 traces, L = 1024, window 5, K = 25 band bins), the reference's
# stages (pipeline.cpp:58-223): remove_dc 2M per trace, detrend_linear 6M per
# trace (two moment sums, then r*slope + intercept subtracted), mean filter
# (2h+1 adds + 1 division) per sample, normalise (1 division per sample + the
# max), radix-2 FFT 5 L log2 L per row (10 ops per butterfly), |X|^2 3 per kept bin.
_M2, _N2, _L2, _W2, _K2 = 512, 1024, 1024, 5, 25
FE_FP64_OPS_PER_RECORD = (8 * _M2 * _N2 + (_W2 + 1) * _M2 * _N2 + 2 * _M2 * _N2 + 5 * _L2 * 10 * _M2
                          + 3 * _K2 * _M2)


def _fp64_peak():
    """fp64 add throughput measured on the box (scripts/micro/fp64peak.cu,
    profiles/r02_fp64_peak.json), else 148 SMs x 64 lanes x 1.965 GHz."""
    import os
    try:
        with open(os.path.join(B.ROOT, "profiles", "r02_fp64_peak.json")) as f:
            d = json.load(f)
        return float(d["dadd_gops"]), "measured (profiles/r02_fp64_peak.json, scripts/micro/fp64peak.cu)"
    except Exception:
        return 148 * 64 * 1.965, "derived (148 SMs x 64 fp64 lanes x 1.965 GHz)"


def run_cfg2(args):
    """Config 2 as a throughput config: a batch of raw fp32
    records through the batched device detect() (front end writing each band
    map straight into the CFAR input, one CFAR call for the batch); the
    single-record host detect() latency is reported beside it."""
    import torch
    import paper_2012_11077_b200 as uwb
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import DetectBatch, kernel_launches
    world, rank, dist = _init_dist()
    n_all, M, Nn = 1024, 512, 1024
    m0, m1 = rank * n_all // world, (rank + 1) * n_all // world
    recs = torch.stack([synth.cfg2_record(seed=2 + i, device="cuda") for i in range(m0, m1)]).contiguous()
    config = uwb.PipelineConfig(mean_filter_window=5, fft_length=1024, band_low_hz=0.3, band_high_hz=0.8,
                                cfar=uwb.CfarParams(1, 4, 1e-3))
    db = DetectBatch(m1 - m0, M, Nn, config, prf=20.0, dtype=torch.float32, det_capacity=2048)
    sampler = B.ClockSampler(torch.cuda.current_device())
    sampler.start()
    l0 = kernel_launches()
    from paper_2012_11077_b200.batch import phase_ms4
    phase_ms4(1024)
    ms = _events_time(lambda: db(recs, phase_events=True), args.steps, args.warmup, world, dist)
    launches = (kernel_launches() - l0) * args.steps // (args.steps + args.warmup)
    clocks = sampler.stop()
    db.check_inputs()
    # the front end's share of the step: step time minus the CFAR call's phases
    ph = _phases(args.steps)
    cfar_ms = sum(ph.values()) if ph else 0.0
    fe_ms = ms - cfar_ms
    n_loc = m1 - m0
    ops = FE_FP64_OPS_PER_RECORD * n_loc
    peak_fp64, peak_src = _fp64_peak()
    fe_roof = {"bound": "fp64", "kernel": "frontend_stats_kernel + frontend_fft1024_kernel",
               "achieved": ops / (fe_ms / 1e3) / 1e9, "peak": peak_fp64, "unit": "Gop/s (fp64 add/mul)",
               "frac": ops / (fe_ms / 1e3) / 1e9 / peak_fp64, "traffic": None,
               "ops_per_record": FE_FP64_OPS_PER_RECORD, "launch_ms": fe_ms, "peak_source": peak_src,
               "timing": "front end = step (CUDA events) minus the CFAR call's phase events",
               "hbm_frac": (n_loc * (M * Nn * 4 + M * db.kept * 8)) / (fe_ms / 1e3) / 1e9 / B._peaks()[0],
               "cfar_phases_ms": ph}
    # end to end: pinned host batch -> H2D -> detect -> D2H of masks and counts
    host = torch.empty(recs.shape, dtype=torch.float32, pin_memory=True)
    host.copy_(recs)
    dev_in = torch.empty_like(recs)
    mask_host = torch.empty(db.mask_bits.shape, dtype=torch.int32, pin_memory=True)
    cnt_host = torch.empty(db.counts.shape, dtype=torch.int64, pin_memory=True)

    def e2e_step():
        dev_in.copy_(host, non_blocking=True)
        db(dev_in)
        mask_host.copy_(db.mask_bits, non_blocking=True)
        cnt_host.copy_(db.counts, non_blocking=True)
        torch.cuda.synchronize()

    e2e_step()
    t0 = time.perf_counter()
    for _ in range(max(args.e2e_steps, 1)):
        e2e_step()
    e_ms = torch.tensor([(time.perf_counter() - t0) * 1e3 / max(args.e2e_steps, 1)], dtype=torch.float64,
                        device="cuda")
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e_ms = float(e_ms.item())
    # single-record latency through the host-level detect() drop-in
    rec0 = recs[0].double().cpu().numpy()
    frame = uwb.RadarFrame(rec0, fast_rate=39e9, prf=20.0)
    uwb.detect(frame, config)
    t0 = time.perf_counter()
    for _ in range(5):
        uwb.detect(frame, config)
    host_ms = (time.perf_counter() - t0) * 1e3 / 5
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        from oracle.pyoracle import RefLib
        ref = RefLib()
        kw = dict(fast_rate=39e9, prf=20.0, mean_filter_window=5, fft_length=1024, guard_radius=1,
                  background_radius=4, pfa=1e-3)
        ref.detect(rec0, **kw)
        t0 = time.perf_counter()
        for _ in range(5):
            ref.detect(rec0, **kw)
        secs = (time.perf_counter() - t0) / 5
        cpu = {"value": 1.0 / secs, "unit": "records/s", "cores": 1, "kind": "reference",
               "sample": f"one config-2 record through uwbvital_ref::detect (FFT: the FFTW-API shim, not FFTW), "
                         f"{secs * 1e3:.1f} ms"}
    if rank == 0:
        _line(metric="front end + CA-CFAR records/s (detect(), config 2)", value=n_all / (ms / 1e3),
              unit="records/s", n_gpus=world, steps=args.steps, warmup=args.warmup, ms_per_step=ms,
              config={"workload": f"cfg2 records batched: {n_all} raw fp32 records 512x1024 at 20 Hz -> DC, "
                                  "detrend, mean filter 5, normalise, FFT L=1024, band 0.3-0.8 Hz (K=25), CFAR g1 b4 "
                                  "Pfa 1e-3 (uwb_dev_detect_batch)",
                      "band_bins": db.kept, "parallelism": f"dp{world} (records sharded)",
                      "single_record_host_detect_ms": host_ms},
              roofline=fe_roof, cpu_baseline=cpu,
              e2e={"value": n_all / (e_ms / 1e3), "unit": "records/s",
                   "h2d_bytes_per_step": int(host.numel() * 4) * world,
                   "d2h_bytes_per_step": int(mask_host.numel() * 4 + cnt_host.numel() * 8) * world,
                   "ms_per_step": e_ms, "timer": "host wall clock, H2D + detect + D2H"},
              gpu_launches=int(launches), clocks=clocks)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------ Table I --
TABLE1 = [(4, 8), (4, 12), (8, 8), (8, 12)]


def run_table1(args):
    """The paper's Table I on one 1024 x 600 fp64 map: naive
    ring-sum CA-CFAR vs the integral-image CA-CFAR, same mask, on the GPU
    (device-resident map, CUDA events) and with the reference on one host core
    (uwbvital_ref::cfar2d_naive / cfar2d_integral, threads=1)."""
    import torch
    import paper_2012_11077_b200 as uwb
    from paper_2012_11077_b200 import synth
    from paper_2012_11077_b200.batch import BatchCfar
    from oracle.pyoracle import RefLib
    world, rank, dist = _init_dist()
    R, C, pfa = 1024, 600, 1e-4
    m = synth.exponential_maps(1, R, C, seed=77, dtype=torch.float64, device="cuda")
    host = m[0].cpu().numpy()
    ref = None if args.no_cpu_baseline else RefLib()
    table = []
    for g, b in TABLE1:
        # both backends write bit masks and sorted lists (no per-cell u8 mask, so
        # neither is slowed by byte-per-cell output the paper's timing does not have)
        runner = BatchCfar(1, R, C, uwb.CfarParams(g, b, pfa), torch.float64, det_capacity=1 << 14)
        ii = _events_time(lambda: runner(m), args.steps, args.warmup, world, dist)
        mask_ii = runner.mask_bits[0].clone()
        nv = _events_time(lambda: runner(m, naive=True), args.steps, args.warmup, world, dist)
        same = bool(torch.equal(mask_ii, runner.mask_bits[0]))
        row = {"guard": g, "train": b, "gpu_naive_ms": nv, "gpu_integral_ms": ii, "gpu_speedup": nv / ii,
               "masks_equal": same}
        if ref is not None:
            t0 = time.perf_counter()
            ref.cfar2d(host, g, b, pfa, "naive")
            t1 = time.perf_counter()
            ref.cfar2d(host, g, b, pfa, "integral")
            t2 = time.perf_counter()
            row.update({"cpu_naive_ms": (t1 - t0) * 1e3, "cpu_integral_ms": (t2 - t1) * 1e3,
                        "cpu_speedup": (t1 - t0) / (t2 - t1)})
        table.append(row)
    if rank == 0:
        _line(metric="Table I (PAPER.md:77-81): naive / integral-image CA-CFAR time ratio, 1024x600 fp64",
              value=min(r["gpu_speedup"] for r in table), unit="x (min over rows)", steps=args.steps,
              warmup=args.warmup, ms_per_step=None,
              config={"workload": "one Exp(1) fp64 map 1024 x 600, Pfa 1e-4, (guard, train) per PAPER.md Table I",
                      "spec": "II >= 2x naive on every row (SPEC.md:483-484)"},
              table=table, cpu_baseline=None, e2e=None, roofline=None, gpu_launches=None, clocks=None)
    return 0


def run_reference_cfg(args):
    """--impl reference for configs 4/5/1/2: the reference CPU path on the host cores."""
    world, rank, _ = B._dist()
    if rank != 0:
        return 0
    import torch
    from oracle.pyoracle import OracleLib, RefLib
    from paper_2012_11077_b200 import synth
    cores = B._cpu_threads()
    ref = RefLib()
    if args.config == 4:
        m = synth.cfg4_map(seed=4, device="cpu", rows=4096, cols=16384).numpy()[None]
        times = [ref.time_cfar_batch(m, 4, 32, 1e-5, 1, ref_threads=cores)[0] for _ in range(args.steps)]
        cells, what = m[0].size, f"4096 of the 16384 rows of the config-4 map per step, cfar2d_integral(threads={cores})"
    elif args.config == 5:
        o = OracleLib()
        m = synth.cfg5_maps(1, seed=5_000, device="cpu", rows=8192, cols=2048)[0].double().numpy()
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            for (gr, gc, br, bc), pfa in CFG5_RUNS:
                o.cfar(m, gr, gc, br, bc, pfa)
            times.append(time.perf_counter() - t0)
        cells, what = 4 * m.size, "one config-5 map x 4 runs, C restatement (reference has no per-axis windows)"
        cores = 1
    elif args.config == 1:
        m = synth.cfg1_map(seed=1, device="cpu").numpy()
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            ref.cfar2d(m, 2, 8, 1e-4)
            times.append(time.perf_counter() - t0)
        cells, what, cores = m.size, "the config-1 map, cfar2d_integral(threads=1)", 1
    else:
        rec = synth.cfg2_record(seed=2, device="cpu").double().numpy()
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            ref.detect(rec, fast_rate=39e9, prf=20.0, mean_filter_window=5, fft_length=1024, guard_radius=1,
                       background_radius=4, pfa=1e-3)
            times.append(time.perf_counter() - t0)
        step = statistics.mean(times)
        _line(impl="reference", metric="front end + CA-CFAR records/s (detect(), config 2)", value=1.0 / step,
              unit="records/s", steps=args.steps, warmup=args.warmup, ms_per_step=step * 1e3,
              config={"workload": "cfg2 record through uwbvital_ref::detect (FFTW-API shim)"},
              cpu_baseline={"value": 1.0 / step, "unit": "records/s", "cores": 1, "kind": "reference",
                            "sample": "one config-2 record per step"},
              e2e={"value": 1.0 / step, "unit": "records/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        return 0
    step = statistics.mean(times)
    v = cells / step / 1e9
    _line(impl="reference", metric=B.METRIC, value=v, unit=B.UNIT, steps=args.steps, warmup=args.warmup,
          ms_per_step=step * 1e3, config={"workload": f"config {args.config}", "sample": what},
          cpu_baseline={"value": v, "unit": B.UNIT, "cores": cores, "kind": "reference" if args.config != 5 else "port",
                        "sample": what},
          e2e={"value": v, "unit": B.UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    return 0


def run(args):
    if args.config == 6:
        return run_table1(args)
    if args.impl == "reference":
        return run_reference_cfg(args)
    return {4: run_cfg4, 5: run_cfg5, 1: run_cfg1, 2: run_cfg2}[args.config](args)
