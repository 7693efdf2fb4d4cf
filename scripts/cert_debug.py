"""Debug: cells the certified path misses vs the exact path (config-3 maps)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2012_11077_b200 as uwb
from paper_2012_11077_b200 import synth
from paper_2012_11077_b200.batch import BatchCfar

n = 8
maps = synth.cfg3_maps(n, seed=11, device="cuda")
p = uwb.CfarParams(2, 8, 1e-4)
c = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=1024)
e = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=1024)
c(maps); e(maps, exact=True); torch.cuda.synchronize()
d = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=1024)
d(maps, dense_tables=True); torch.cuda.synchronize()
print("counts cert-dense", d.counts.tolist())
print("counts cert", c.counts.tolist()); print("counts exact", e.counts.tolist())
for i in range(n):
    a, b = c.mask(i), e.mask(i)
    miss = np.argwhere((b == 1) & (a == 0)); extra = np.argwhere((a == 1) & (b == 0))
    for r, cc in miss[:10]:
        print(f"map {i} missed ({r},{cc}) tile ({r//2},{cc//2}) par ({r%2},{cc%2}) band {cc//256} tcol {(cc//2)%128} grp {((cc//2)%128)//8} j {((cc//2)%8)} trow%8 {(r//2)%8}")
    if len(extra): print("extra", extra[:5].tolist())

import math
full = BatchCfar(n, 1024, 1024, p, torch.float32, det_capacity=1024, want_thresholds=True)
full(maps); torch.cuda.synchronize()
def box(a, h0, h1, axis):
    cs = np.cumsum(np.pad(a, [(1,0) if ax==axis else (0,0) for ax in range(a.ndim)]), axis=axis)
    N = a.shape[axis]; idx = np.arange(N)
    lo = np.clip(idx + h0, 0, N); hi = np.clip(idx + h1 + 1, 0, N)
    return np.take(cs, hi, axis=axis) - np.take(cs, lo, axis=axis)
def trng(h, a): return math.ceil((a - h)/2), (a + h - 1)//2
def grng(g, a): return math.ceil((a - g - 1)/2), (a + g)//2
for i in range(n):
    a, b = c.mask(i), e.mask(i)
    for r, cc in np.argwhere((b == 1) & (a == 0))[:3]:
        x = maps[i].double().cpu().numpy()
        T = full.thresholds[i, r, cc].item()
        Z = x.reshape(512, 2, 512, 2).sum(axis=(1, 3))
        ar, bc = r % 2, cc % 2
        o0, o1 = trng(10, ar); g0, g1 = grng(2, ar); p0, p1 = trng(10, bc); q0, q1 = grng(2, bc)
        HO = box(box(Z, o0, o1, 0), p0, p1, 1); HG = box(box(Z, g0, g1, 0), q0, q1, 1)
        LB = (HO - HG)[r // 2, cc // 2]
        ring = box(box(x, -10, 10, 0), -10, 10, 1)[r, cc] - box(box(x, -2, 2, 0), -2, 2, 1)[r, cc]
        print(f"map {i} ({r},{cc}) cut {x[r,cc]:.6f} T {T:.6f} ring {ring:.4f} LB {LB:.4f} alpha/n*LB {9.3130566043946388/416*LB:.4f}")
        I, J = r // 2, cc // 2
        print("tile cuts", x[2*I:2*I+2, 2*J:2*J+2])
