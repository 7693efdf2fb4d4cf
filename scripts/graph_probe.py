"""Config-1 map (one 256x512 fp64 map): direct calls vs a captured CUDA graph."""
import time
import numpy as np
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar

m = synth.cfg1_map(seed=1, device="cuda").unsqueeze(0).contiguous()
p = uwb.CfarParams(2, 8, 1e-4)
r = BatchCfar(1, 256, 512, p, torch.float64, det_capacity=4096)
for _ in range(3):
    r(m)
torch.cuda.synchronize()
ref_mask = r.mask(0).copy()
ref_d = r.detections(0)


def timeit(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


direct = timeit(lambda: r(m))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    r(m)  # warm-up on the capture stream
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    r(m)
g.replay()
torch.cuda.synchronize()
assert np.array_equal(r.mask(0), ref_mask)
assert np.array_equal(r.detections(0), ref_d)
graph = timeit(g.replay)
print(f"direct {direct * 1e3:.1f} us/map  graph {graph * 1e3:.1f} us/map (identical outputs)")
