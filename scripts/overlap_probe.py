"""Does running two half-batches on two streams overlap SAT with CFAR?"""
import time
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar

dev = torch.device("cuda:0")
n = 2048
maps = torch.empty((n, 1024, 1024), dtype=torch.float32, device=dev)
for c in range(n // 64):
    synth.cfg3_maps(64, seed=c, device=dev, out=maps[c * 64:(c + 1) * 64])
params = uwb.CfarParams(2, 8, 1e-4)
full = BatchCfar(n, 1024, 1024, params, torch.float32, det_capacity=512, device=dev)
for parts in (2, 4, 8):
    h = n // parts
    runners = [BatchCfar(h, 1024, 1024, params, torch.float32, det_capacity=512, device=dev) for _ in range(parts)]
    streams = [torch.cuda.Stream() for _ in range(parts)]

    def step_split():
        cur = torch.cuda.current_stream()
        for i, (r, s) in enumerate(zip(runners, streams)):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                r(maps[i * h:(i + 1) * h])
        for s in streams:
            cur.wait_stream(s)

    for name, fn in (("serial full batch", lambda: full(maps)), (f"{parts} streams", step_split)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name}: {e0.elapsed_time(e1) / 5:.3f} ms per {n} maps", flush=True)
    del runners
    torch.cuda.empty_cache()
