"""Probe host<->device copy rates on the box (pinned, chunk sizes, streams)."""
import time
import torch

dev = torch.device("cuda:0")
GB = 1 << 30
tot = 8 * GB
host = torch.empty(tot // 4, dtype=torch.float32, pin_memory=True)
host.fill_(1.0)
d = torch.empty(tot // 4, dtype=torch.float32, device=dev)
for chunk_mb in (64, 256, 512, 2048, 8192):
    n = chunk_mb * (1 << 20) // 4
    for nstreams in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(nstreams)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, o in enumerate(range(0, host.numel(), n)):
            with torch.cuda.stream(streams[i % nstreams]):
                d[o:o + n].copy_(host[o:o + n], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"H2D chunk {chunk_mb:5d} MB streams {nstreams}: {tot / dt / 1e9:6.1f} GB/s", flush=True)
# D2H
t0 = time.perf_counter()
host.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H 8 GiB: {tot / (time.perf_counter() - t0) / 1e9:6.1f} GB/s")
# simultaneous H2D + D2H
h2 = torch.empty(GB // 4, dtype=torch.float32, pin_memory=True)
d2 = torch.empty(GB // 4, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(host, non_blocking=True)
with torch.cuda.stream(s2):
    for _ in range(4):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D 8 GiB || D2H 4 GiB: {(tot + 4 * GB) / (time.perf_counter() - t0) / 1e9:6.1f} GB/s total")
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max", "--format=csv"], capture_output=True, text=True).stdout)
print(subprocess.run(["bash", "-c", "lscpu | head -20; numactl -H 2>/dev/null | head; nvidia-smi topo -m"], capture_output=True, text=True).stdout)
