#!/usr/bin/env python
"""Benchmark of the north-star path on B200 (BASELINE.json metric).

Metric: CA-CFAR Gcells/s (integral-image backend, reference-exact global SAT)
with the achieved-HBM roofline fraction of the dominant kernel, beside the
reference's CPU implementation.

Workload (N=1 line): BASELINE.json config 3 - 4096 independent fp32 maps of
1024 x 1024, Exp(1) background + 32 seeded targets at U(8,20) dB each, guard 2,
training 8, Pfa 1e-4. One step = SAT (kernel c) + CFAR threshold / bit mask /
detection compaction (kernel d) + per-map detection sort over the whole batch.
The batch (16 GiB of input per pass) is far larger than the 126 MB L2, so no
explicit flush is needed between steps.

Launch: ``python bench.py [--gpus N --steps K --warmup W]``; for N > 1 under
``torch.distributed.run`` (one rank per GPU, NCCL); the 4096 maps are sharded
in 64-map blocks across ranks (strong scaling) and each step ends with the
detection-count all-reduce. ``--impl reference`` times the reference C++ code
(oracle/_ref, compiled from /root/reference) on the host cores instead.
``--config {1,2,4,5}`` measures the other BASELINE.json configurations
(bench_configs.py) with the same JSON schema.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_MAPS = 4096
ROWS = COLS = 1024
GUARD, TRAIN, PFA = 2, 8, 1e-4
CHUNK = 64  # maps per generator block (sharding granularity)
SEED = 3
METRIC = "CA-CFAR Gcells/s (integral image, exact fp64 SAT) + achieved HBM fraction"
UNIT = "Gcells/s"
WORKLOAD = ("cfg3: 4096 fp32 maps 1024x1024, Exp(1) + 32 targets/map at U(8,20) dB, guard 2, "
            "train 8, Pfa 1e-4, border Clamp, ties H0")
SAT_BYTES_PER_CELL = 4 + 8        # read fp32 cell, write fp64 table entry
CFAR_BYTES_PER_CELL = 8 + 4 + 1 / 8  # read table entry + CUT, write mask bit
FUSED_BYTES_PER_CELL = 4 + 1 / 8     # fused SAT+CFAR: read fp32 cell once, write mask bit
CERT_BYTES_PER_CELL = 4              # certify: read fp32 cell once (candidates ~1e-4 of cells)
SPARSE_SAT_BYTES_PER_CELL = 4        # sparse SAT: read fp32 cell once (writes ~8 taps x 32 B per candidate)
RESOLVE_BYTES_PER_CELL = 1 / 8       # resolve: mask bit per cell (taps and lists ~Pfa of the cells)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.lines: list[str] = []
        self._t = None

    def start(self):
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.idx).uuid)
            sel = ["-i", "GPU-" + uuid if not uuid.startswith("GPU-") else uuid]
        except Exception:
            sel = ["-i", str(self.idx)]
        try:
            self.proc = subprocess.Popen(["nvidia-smi", *sel, f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self._t:
            self._t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _init_rank(world: int, local: int):
    """One process per GPU over NCCL. UWB_DIST_BACKEND=gloo (test hook) lets
    several ranks share the visible GPUs to exercise the multi-rank code path
    (no kernel of one rank waits on another rank)."""
    import torch
    import torch.distributed as dist
    idx = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(idx)
    if world > 1:
        backend = os.environ.get("UWB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", idx))
        else:
            dist.init_process_group(backend)
    return torch.device("cuda", idx)


def _shard(world: int, rank: int):
    """Contiguous blocks of 64-map chunks per rank (maps are independent units;
    shard.map_shard)."""
    from paper_2012_11077_b200.shard import map_shard
    return map_shard(N_MAPS, world, rank, block=CHUNK)


def _generate(m0: int, m1: int, device):
    import torch
    from paper_2012_11077_b200 import synth
    maps = torch.empty((m1 - m0, ROWS, COLS), dtype=torch.float32, device=device)
    for c in range(m0 // CHUNK, m1 // CHUNK):
        i = c * CHUNK - m0
        synth.cfg3_maps(CHUNK, seed=SEED * 1_000_003 + c, device=device, out=maps[i:i + CHUNK])
    return maps


def _cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _cpu_name() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def reference_cells_per_s(maps_host, budget_s: float = 12.0, max_maps: int = 512):
    """Times the reference cfar2d_integral (oracle/_ref, compiled from
    /root/reference) map-parallel on all host threads, threads=1 per map
    (SURVEY 8d way ii); input widening excluded from the timer (bench.hpp:70-72)."""
    import numpy as np
    from oracle.pyoracle import RefLib
    ref = RefLib()
    cores = _cpu_threads()
    one, _ = ref.time_cfar_batch(np.ascontiguousarray(maps_host[:1]), GUARD, TRAIN, PFA, 1)
    n = int(max(cores, min(max_maps, len(maps_host), budget_s * cores / max(one, 1e-3))))
    n = min(n, len(maps_host))
    secs, counts = ref.time_cfar_batch(np.ascontiguousarray(maps_host[:n]), GUARD, TRAIN, PFA, cores)
    cells = n * ROWS * COLS
    return cells / secs, {"maps": n, "seconds": secs, "cores": cores, "one_map_1thread_s": one,
                          "detections": int(counts.sum())}


def _load_synth():
    """The seeded generators (paper_2012_11077_b200/synth.py, torch only) loaded
    by path, so the reference arm never imports the product package (whose
    __init__ loads libuwbvital_b200.so)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_uwb_synth_standalone", os.path.join(ROOT, "paper_2012_11077_b200", "synth.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


REF_MAPS_PER_STEP = 512


def run_reference(args):
    """The reference's own CPU path (oracle/_ref = /root/reference/proj/src
    compiled unchanged): cfar2d_integral per map, map-parallel on every host
    thread (SURVEY 8d way ii), on a bounded sample of config 3 per step. Also
    reports, once, way (i): one map at a time with the reference's own row
    split over all threads (cfar.cpp:142-161)."""
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    import numpy as np
    synth = _load_synth()
    from oracle.pyoracle import RefLib
    cores = _cpu_threads()
    n = max(cores, min(N_MAPS, REF_MAPS_PER_STEP))
    maps = np.empty((n, ROWS, COLS), dtype=np.float32)
    for c in range(0, n, CHUNK):  # the same generator blocks as the device arm's first maps
        k = min(CHUNK, n - c)
        maps[c:c + k] = synth.cfg3_maps(CHUNK, seed=SEED * 1_000_003 + c // CHUNK, device="cpu")[:k].numpy()
    ref = RefLib()
    for _ in range(args.warmup):
        ref.time_cfar_batch(maps[:cores], GUARD, TRAIN, PFA, cores)
    times = []
    for _ in range(args.steps):
        secs, counts = ref.time_cfar_batch(maps, GUARD, TRAIN, PFA, cores)
        times.append(secs)
    step = statistics.mean(times)
    value = n * ROWS * COLS / step / 1e9
    k_rows = min(8, n)
    secs_rows, _ = ref.time_cfar_batch(maps[:k_rows], GUARD, TRAIN, PFA, 1, cores)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": max(world, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, config 3)",
        "config": {"workload": WORKLOAD, "sample_maps_per_step": n, "parallelism": f"{cores} host threads",
                   "detections_per_step": int(counts.sum())},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{n} config-3 maps per step (the device arm's maps 0..{n - 1}), "
                                   f"uwbvital_ref::cfar2d_integral(map, params, 1) map-parallel on {cores} threads "
                                   f"({_cpu_name()})",
                         "row_split_value": k_rows * ROWS * COLS / secs_rows / 1e9,
                         "row_split_sample": f"{k_rows} maps one at a time, cfar2d_integral(map, params, {cores}) "
                                             f"(the reference's own row split, cfar.cpp:142-161)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def step_kernels(cert_ms: float, sat_ms: float, cfar_ms: float, cells: float, certified: bool, fused: bool = False):
    """{kernel: (ms per launch, algorithmic bytes per launch)} of one CFAR call
    from its phase times (batch.phase_ms4). Certified path: cert_kernel and the
    sparse SAT each read the map once; the resolve writes the mask bits (its
    taps and lists are ~Pfa of the cells). Exact path: the SAT writes the fp64
    table, the ring CFAR reads it back with the CUT. Fused: one map read."""
    if fused:
        return {"cfar_fused_kernel": (cfar_ms, FUSED_BYTES_PER_CELL * cells)}
    if certified:
        return {"cert_kernel": (cert_ms, CERT_BYTES_PER_CELL * cells),
                "sat_systolic_kernel(sparse)": (sat_ms, SPARSE_SAT_BYTES_PER_CELL * cells),
                "cert_resolve_kernel": (cfar_ms, RESOLVE_BYTES_PER_CELL * cells)}
    return {"sat_systolic_kernel": (sat_ms, SAT_BYTES_PER_CELL * cells),
            "cfar_ws_kernel": (cfar_ms, CFAR_BYTES_PER_CELL * cells)}


def roofline_of(kernels: dict, peak: float, peak_src: str) -> dict:
    """Roofline entry of the dominant (longest) kernel of `kernels`."""
    dom = max(kernels, key=lambda k: kernels[k][0])
    ms, by = kernels[dom]
    ach = by / (ms / 1e3) / 1e9 if ms > 0 else 0.0
    ncu = _ncu_traffic() or {}
    return {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "traffic": None, "traffic_source": None, "bytes_per_cell": None, "launch_ms": ms,
            "launch_bytes": by, "peak_source": peak_src,
            "ncu_kernels_known": sorted(ncu.keys())}


def _ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2012_11077_b200 as uwb
    from paper_2012_11077_b200.batch import BatchCfar, host_cfar2d_batch, kernel_launches, phase_ms4

    world, rank, local = _dist()
    dev = _init_rank(world, local)
    m0, m1 = _shard(world, rank)
    n_local = m1 - m0
    maps = _generate(m0, m1, dev)
    params = uwb.CfarParams(GUARD, TRAIN, PFA)
    det_cap = 512
    runner = BatchCfar(n_local, ROWS, COLS, params, torch.float32, det_capacity=det_cap, device=dev)
    total_count = torch.zeros(1, dtype=torch.int64, device=dev)

    def step(phase=False):
        runner(maps, phase_events=phase, fused=args.fused, exact=args.exact)
        total_count.copy_(runner.counts.sum().view(1))
        if world > 1:
            dist.all_reduce(total_count)  # final detection-count reduce (NCCL)

    def barrier():
        if world > 1:
            dist.barrier()

    for i in range(max(args.warmup, 0)):
        step(phase=(i == args.warmup - 1))  # the last warm-up also creates the phase events
    torch.cuda.synchronize()
    runner.check_inputs()
    phase_ms4(1024)  # clear the ring

    sampler = ClockSampler(dev.index)
    sampler.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    launches0 = kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step(phase=True)
    ev1.record()
    torch.cuda.synchronize()
    barrier()
    launches = kernel_launches() - launches0
    clocks = sampler.stop()
    ms_local = ev0.elapsed_time(ev1)
    ms_t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    ms_per_step = ms / args.steps
    cells_total = N_MAPS * ROWS * COLS
    value = cells_total / (ms_per_step / 1e3) / 1e9

    ph = phase_ms4(1024)
    cert_ms, sat_ms, cfar_ms, sort_ms = (float(np.mean(ph[:, i])) for i in range(4)) if len(ph) else (0.0,) * 4
    peak, peak_src = _peaks()
    cells_local = n_local * ROWS * COLS
    certified = cert_ms > 0.02 * (sat_ms + cfar_ms + 1e-9) and not args.exact and not args.fused
    # whole-map batches run SAT + CFAR as one kernel (cfar_fused.cu); its phase
    # is "cfar" and the "sat" phase is empty
    fused = args.fused and cfar_ms > 0 and sat_ms < 0.02 * cfar_ms
    if fused:
        kernels = {"cfar_fused_kernel": (cfar_ms, FUSED_BYTES_PER_CELL * cells_local)}
    elif certified:
        # certified-decision path (DESIGN 4c): cert_kernel reads the map once
        # (window sums of quantised cells -> candidate list), the SAT reads it
        # again and stores only the candidates' taps, the resolve reads ~Pfa of
        # the cells' taps; algorithmic bytes per cell = one map read per pass
        kernels = {
            "cert_kernel": (cert_ms, CERT_BYTES_PER_CELL * cells_local),
            "sat_systolic_kernel(sparse)": (sat_ms, SPARSE_SAT_BYTES_PER_CELL * cells_local),
            "cert_resolve_kernel": (cfar_ms, RESOLVE_BYTES_PER_CELL * cells_local),
        }
    else:
        kernels = {
            "sat_systolic_kernel": (sat_ms, SAT_BYTES_PER_CELL * cells_local),
            "cfar_ws_kernel": (cfar_ms, CFAR_BYTES_PER_CELL * cells_local),
        }
    dom = max(kernels, key=lambda k: kernels[k][0])
    dom_ms, dom_bytes = kernels[dom]
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
    step_bytes = sum(v[1] for v in kernels.values())
    ncu = _ncu_traffic() or {}
    traffic = ncu.get(dom, {}).get("dram_bytes_per_launch_per_map")
    traffic = traffic * n_local if traffic else None
    traffic_src = ncu.get(dom, {}).get("source") if traffic else None

    # ---- end to end through the public host API: pinned host maps -> H2D -> SAT+CFAR+sort -> D2H
    e2e = None
    if not args.no_e2e:
        host_maps = torch.empty((n_local, ROWS, COLS), dtype=torch.float32, pin_memory=True)
        host_maps.copy_(maps)
        bits = torch.zeros((n_local, ROWS, (COLS + 31) // 32), dtype=torch.int32, pin_memory=True)
        dets = torch.zeros((n_local, det_cap, 32), dtype=torch.uint8, pin_memory=True)
        counts = torch.zeros(n_local, dtype=torch.int64, pin_memory=True)
        host_cfar2d_batch(host_maps, params, bits, dets, counts, det_cap, maps_per_chunk=args.e2e_chunk)
        e_steps = max(2, min(args.steps, args.e2e_steps))
        barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            host_cfar2d_batch(host_maps, params, bits, dets, counts, det_cap, maps_per_chunk=args.e2e_chunk)
        t1 = time.perf_counter()
        barrier()
        e_ms = torch.tensor([(t1 - t0) * 1e3 / e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e_ms_v = float(e_ms.item())
        same = bool(torch.equal(counts, runner.counts.cpu()))
        e2e = {"value": cells_total / (e_ms_v / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(host_maps.numel() * 4) * world,
               "d2h_bytes_per_step": int(bits.numel() * 4 + dets.numel() + counts.numel() * 8) * world,
               "ms_per_step": e_ms_v, "steps": e_steps, "maps_per_chunk": args.e2e_chunk,
               "timer": "host wall clock around the synchronous call",
               "matches_device_path": same}
        del host_maps

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = maps[: min(512, n_local)].cpu().numpy()
        v, info = reference_cells_per_s(sample)
        cpu = {"value": v / 1e9, "unit": UNIT, "cores": info["cores"], "kind": "reference",
               "sample": f"{info['maps']} config-3 maps, uwbvital_ref::cfar2d_integral map-parallel on "
                         f"{info['cores']} threads ({_cpu_name()}), {info['seconds']:.2f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator for BASELINE config 3, device-resident fp32 input)",
            "config": {"workload": WORKLOAD, "n_maps": N_MAPS, "rows": ROWS, "cols": COLS,
                       "input_dtype": "f32", "sat_mode": "global (bit-identical to the reference)",
                       "kernels": ("fused SAT+CFAR (flags bit 4)" if args.fused else
                                   "certify (cert_kernel + cert_mark_kernel) + sparse SAT (sat_systolic_kernel) "
                                   "+ resolve (cert_resolve_kernel) + sort" if certified else
                                   "SAT (sat_systolic_kernel) + CFAR (cfar_ws_kernel) + sort"),
                       "decision": ("certified: cells whose exact-arithmetic lower bound of T exceeds the CUT "
                                    "are decided without the table; the rest are resolved from exact fp64 SAT "
                                    "taps (bit-identical to the reference)" if certified else "exact"),
                       "l2": "inputs 16 GiB per pass >> 126 MB L2 (no flush needed)",
                       "parallelism": f"dp{world} (maps sharded in 64-map blocks)",
                       "detections_per_step": int(total_count.item()) if world > 1 else
                       int(runner.counts.sum().item())},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "bytes_per_cell": dom_bytes / cells_local,
                         "launch_ms": dom_ms, "peak_source": peak_src,
                         **({"note": "fused SAT+CFAR: the table stays in shared memory, so HBM carries only "
                                     "the map read and the mask; the kernel is bound by the SAT wavefront "
                                     "(one dependent fp64 chain per 128-column band, 3 bands per SM), see "
                                     "DESIGN.md 4(e)"} if fused else {})},
            "phases_ms": {"certify": cert_ms, "sat": sat_ms, "cfar": cfar_ms, "sort": sort_ms},
            # whole-step HBM fraction against the algorithmic bytes of the kernels above
            "step_hbm_frac": step_bytes / (ms_per_step / 1e3) / 1e9 / peak,
            # HBM fraction the two-pass algorithm (table written and read back) would need for this time
            "two_pass_equiv_hbm_frac": (SAT_BYTES_PER_CELL + CFAR_BYTES_PER_CELL) * cells_local
                                       / (ms_per_step / 1e3) / 1e9 / peak,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _ensure_world(args):
    """--gpus N is honoured: under torch.distributed.run WORLD_SIZE must equal N;
    without it, N > 1 re-executes this command under torch.distributed.run (one
    rank per GPU), after checking that N devices are visible. The reference arm
    runs on the host cores (rank 0 only) and needs no ranks."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus < 1:
        print(json.dumps({"error": f"--gpus {args.gpus} < 1"}), flush=True)
        return 2
    if args.impl == "reference" or world == args.gpus:
        return None
    if world != 1:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        return 2
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and os.environ.get("UWB_DIST_BACKEND", "nccl") == "nccl":
        print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s) visible"}), flush=True)
        return 2
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunk", type=int, default=64, help="maps per H2D chunk in the end-to-end call")
    ap.add_argument("--maps", type=int, default=N_MAPS, help="batch size (profiling runs only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--fused", action="store_true",
                    help="device path through the fused SAT+CFAR kernel (flags bit 4) instead of SAT + ring CFAR")
    ap.add_argument("--exact", action="store_true",
                    help="device path through the exact two-kernel path (full fp64 table + ring CFAR)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5, 6],
                    help="BASELINE.json configuration (3 = the headline line; 6 = the paper's Table I; "
                         "see bench_configs.py)")
    args = ap.parse_args()
    globals()["N_MAPS"] = args.maps
    rc = _ensure_world(args)
    if rc is not None:
        return rc
    if args.config != 3:
        import bench_configs
        return bench_configs.run(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
