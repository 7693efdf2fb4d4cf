"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference measures nothing on a public dataset; BASELINE.json
defines every workload synthetically and these generators follow those
definitions (shapes, distributions, SNR conventions of SURVEY 8d: "X dB SNR"
adds 10^(X/10) times the reference power to the cell). They run with torch on
any device; the same bytes are handed to the GPU path and (after a copy) to the
CPU oracle. Input generation is never inside a timed region.
"""
from __future__ import annotations

import math

import torch

CONFIGS = {
    1: dict(name="cfg1_single_fp64_256x512", rows=256, cols=512, n_maps=1, dtype=torch.float64,
            guard=(2, 2), train=(8, 8), pfa=1e-4),
    2: dict(name="cfg2_frontend_512x1024", m=512, n=1024, prf=20.0, window=5, band=(0.3, 0.8),
            guard=(1, 1), train=(4, 4), pfa=1e-3),
    3: dict(name="cfg3_batched_4096x1024x1024_fp32", rows=1024, cols=1024, n_maps=4096,
            dtype=torch.float32, guard=(2, 2), train=(8, 8), pfa=1e-4),
    4: dict(name="cfg4_single_16384x16384_fp32", rows=16384, cols=16384, n_maps=1,
            dtype=torch.float32, guard=(4, 4), train=(32, 32), pfa=1e-5),
    5: dict(name="cfg5_kclutter_64x8192x2048_fp32", rows=8192, cols=2048, n_maps=64,
            dtype=torch.float32,
            windows=[((1, 3), (4, 16)), ((3, 1), (16, 4))], pfas=[1e-3, 1e-5]),
}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def exponential_maps(n_maps: int, rows: int, cols: int, seed: int, dtype=torch.float32, device="cuda",
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """i.i.d. Exp(1) cells (|CN(0,1)|^2)."""
    g = _gen(seed, device)
    x = out if out is not None else torch.empty((n_maps, rows, cols), dtype=dtype, device=device)
    x.exponential_(1.0, generator=g)
    return x


def add_point_targets(maps: torch.Tensor, per_map: int, snr_db_lo: float, snr_db_hi: float, seed: int,
                      extent: int = 1) -> torch.Tensor:
    """Adds `per_map` targets at seeded distinct positions per map; each covers an
    extent x extent block whose cells all get += 10^(snr/10) (unit background)."""
    n_maps, rows, cols = maps.shape
    dev = maps.device
    g = _gen(seed + 7919, dev)
    R, Cc = rows - extent + 1, cols - extent + 1
    # distinct top-left positions per map (sampling without replacement by rank),
    # 64 maps at a time to bound the key buffer
    if R * Cc <= 1 << 22:
        pos = torch.cat([torch.topk(torch.rand((min(64, n_maps - i), R * Cc), generator=g, device=dev),
                                    per_map, dim=1).indices for i in range(0, n_maps, 64)])
    else:
        pos = torch.randint(0, R * Cc, (n_maps, per_map), generator=g, device=dev)
    snr = snr_db_lo + (snr_db_hi - snr_db_lo) * torch.rand((n_maps, per_map), generator=g, device=dev,
                                                           dtype=torch.float64)
    amp = torch.pow(10.0, snr / 10.0).to(maps.dtype)
    r0 = pos // Cc
    c0 = pos % Cc
    mi = torch.arange(n_maps, device=dev).unsqueeze(1).expand_as(pos)
    for dr in range(extent):
        for dc in range(extent):
            maps.index_put_((mi.reshape(-1), (r0 + dr).reshape(-1), (c0 + dc).reshape(-1)), amp.reshape(-1),
                            accumulate=True)
    return maps


def cfg1_map(seed: int = 1, device="cuda") -> torch.Tensor:
    x = exponential_maps(1, 256, 512, seed, torch.float64, device)
    return add_point_targets(x, 5, 15.0, 15.0, seed)[0]


def cfg3_maps(n_maps: int = 4096, seed: int = 3, device="cuda", out=None) -> torch.Tensor:
    x = exponential_maps(n_maps, 1024, 1024, seed, torch.float32, device, out=out)
    return add_point_targets(x, 32, 8.0, 20.0, seed)


def cfg4_map(seed: int = 4, device="cuda", rows: int = 16384, cols: int = 16384) -> torch.Tensor:
    x = exponential_maps(1, rows, cols, seed, torch.float32, device)
    return add_point_targets(x, 1000, 6.0, 18.0, seed, extent=3)[0]


def _box_mean(tex: torch.Tensor, box: int) -> torch.Tensor:
    """Mean of tex over a box x box window anchored at (r - box/2, c - box/2),
    clamped to the map (edge windows average the cells inside)."""
    rows, cols = tex.shape
    dev = tex.device
    pad = torch.nn.functional.pad(tex.double().cumsum(0).cumsum(1), (1, 0, 1, 0))
    h = box // 2
    ri = torch.arange(rows, device=dev)
    ci = torch.arange(cols, device=dev)
    r0 = (ri - h).clamp(min=0)
    r1 = (ri + box - h).clamp(max=rows)
    c0 = (ci - h).clamp(min=0)
    c1 = (ci + box - h).clamp(max=cols)
    s = pad[r1][:, c1] - pad[r0][:, c1] - pad[r1][:, c0] + pad[r0][:, c0]
    area = ((r1 - r0).unsqueeze(1) * (c1 - c0).unsqueeze(0)).double()
    return (s / area).float()


def cfg5_maps(n_maps: int = 64, seed: int = 5, device="cuda", rows: int = 8192, cols: int = 2048,
              box: int = 16, out: torch.Tensor | None = None) -> torch.Tensor:
    """K-distributed clutter: Gamma(shape 0.5, scale 1) texture, box-averaged
    over 16x16 (window clamped at the map edges: mean of the cells inside),
    times Exp(1) speckle; 64 clusters of 2-6 4-adjacent cells per map, each cell
    += 10^(U(10,25)/10) x the local clutter mean (the smoothed texture at the
    cluster's seed cell). Generated map by map to bound temporary memory."""
    g = _gen(seed, device)
    maps = out if out is not None else torch.empty((n_maps, rows, cols), dtype=torch.float32, device=device)
    steps = [(0, 0), (0, 1), (1, 1), (1, 2), (2, 2), (2, 3)]  # 4-adjacent walk
    n_cl = 64
    for i in range(n_maps):
        tex = torch._standard_gamma(torch.full((rows, cols), 0.5, device=device), generator=g)
        smooth = _box_mean(tex, box)
        del tex
        m = maps[i]
        m.exponential_(1.0, generator=g)
        m.mul_(smooth)
        sr = torch.randint(1, rows - 3, (n_cl,), generator=g, device=device)
        sc = torch.randint(1, cols - 4, (n_cl,), generator=g, device=device)
        sizes = torch.randint(2, 7, (n_cl,), generator=g, device=device)
        snr = 10.0 + 15.0 * torch.rand(n_cl, generator=g, device=device, dtype=torch.float64)
        amp = (torch.pow(10.0, snr / 10.0) * smooth[sr, sc].double()).float()
        for k, (dr, dc) in enumerate(steps):
            use = sizes > k
            m.index_put_(((sr + dr)[use], (sc + dc)[use]), amp[use], accumulate=True)
    return maps


def cfg2_record(seed: int = 2, device="cuda", m: int = 512, n: int = 1024, prf: float = 20.0) -> torch.Tensor:
    """Raw UWB record, fp32 M x N: per-trace (column) DC offset U(-1,1) and linear
    drift slope U(-1e-3,1e-3) along fast time (removed by remove_dc /
    detrend_linear), N(0, 0.1^2) noise, and a respiration target at fast-time bin
    200 (Gaussian range spread sigma 3 bins) modulated 0.5 sin(2 pi 0.4 t + phi)
    with t = n / prf."""
    g = _gen(seed, device)
    dc = torch.rand(n, generator=g, device=device, dtype=torch.float64) * 2 - 1
    slope = (torch.rand(n, generator=g, device=device, dtype=torch.float64) * 2 - 1) * 1e-3
    noise = torch.randn((m, n), generator=g, device=device, dtype=torch.float64) * 0.1
    phi = float(torch.rand(1, generator=g, device=device, dtype=torch.float64).item()) * 2 * math.pi
    mm = torch.arange(m, device=device, dtype=torch.float64).unsqueeze(1)
    tt = torch.arange(n, device=device, dtype=torch.float64).unsqueeze(0) / prf
    target = 0.5 * torch.sin(2 * math.pi * 0.4 * tt + phi) * torch.exp(-((mm - 200.0) ** 2) / (2 * 3.0 ** 2))
    x = dc.unsqueeze(0) + slope.unsqueeze(0) * mm + noise + target
    return x.float()
