"""SAT/CFAR overlap across batch chunks on two streams (config-3 maps)."""
import os
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar

dev = torch.device("cuda:0")
n = int(os.environ.get("MAPS", "4096"))
chunks = int(os.environ.get("CHUNKS", "4"))
maps = torch.empty((n, 1024, 1024), dtype=torch.float32, device=dev)
for c in range(n // 64):
    synth.cfg3_maps(64, seed=c, device=dev, out=maps[c * 64:(c + 1) * 64])
p = uwb.CfarParams(2, 8, 1e-4)
full = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=512, device=dev)
m = n // chunks
parts = [BatchCfar(m, 1024, 1024, p, torch.float32, det_capacity=512, device=dev) for _ in range(chunks)]
prio = int(os.environ.get("PRIO", "0"))
streams = [torch.cuda.Stream(device=dev, priority=(-1 if (prio and i % 2) else 0)) for i in range(2)]


def run_full():
    full(maps)


def run_chunks():
    cur = torch.cuda.current_stream(dev)
    ev = torch.cuda.Event()
    ev.record(cur)
    for i, b in enumerate(parts):
        s = streams[i % 2]
        s.wait_event(ev)
        b(maps[i * m:(i + 1) * m], stream=s)
    for s in streams:
        e = torch.cuda.Event()
        e.record(s)
        cur.wait_event(e)


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print(f"full {timeit(run_full):.2f} ms  chunks={chunks} {timeit(run_chunks):.2f} ms", flush=True)
