"""Where does a bench step's time go outside the SAT/CFAR/sort phases?"""
import time
import torch
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar, phase_ms

dev = torch.device("cuda:0")
n = 1024
maps = torch.empty((n, 1024, 1024), dtype=torch.float32, device=dev)
for c in range(n // 64):
    synth.cfg3_maps(64, seed=c, device=dev, out=maps[c * 64:(c + 1) * 64])
params = uwb.CfarParams(2, 8, 1e-4)
runner = BatchCfar(n, 1024, 1024, params, torch.float32, det_capacity=512, device=dev)
for _ in range(3):
    runner(maps)
torch.cuda.synchronize()
phase_ms(1024)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for phase in (False, True):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    for _ in range(5):
        runner(maps, phase_events=phase)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"phase_events={phase}: device {e0.elapsed_time(e1) / 5:.3f} ms/step, host submit {(t1 - t0) * 1e3 / 5:.3f} ms/step,"
          f" wall {(t2 - t0) * 1e3 / 5:.3f}")
    if phase:
        print(phase_ms(1024))
