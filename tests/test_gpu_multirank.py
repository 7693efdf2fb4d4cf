"""Executed multi-rank runs of the product path on the one-GPU lease.

The reference's only parallel split is the row split of run_cfar, whose output
is bit-identical to the sequential run (/root/reference/proj/src/cfar.cpp:142-161,
proj/tests/test_cfar.cpp:308-320). The B200 path shards whole maps across
ranks (configs 3/5) and rows with a g+b halo (config 4); here N processes share
cuda:0 (UWB_DIST_BACKEND=gloo: no kernel of one rank waits on another, the
count all-reduce goes through gloo) and run scripts/multirank_check.py, i.e.
bench.py's own shard, generator and count reduce. The concatenated per-rank
outputs must equal the world-1 run bit for bit, and the reduced totals must
equal the sum of the per-rank counts."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, out):
    env = dict(os.environ, UWB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "scripts", "multirank_check.py"), "--out", str(out)]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [dict(np.load(os.path.join(out, f"rank{k}.npz"), allow_pickle=False)) for k in range(world)]


@pytest.fixture(scope="module")
def world1(tmp_path_factory):
    return _run(1, tmp_path_factory.mktemp("w1"))


@pytest.mark.parametrize("world", [2, 4])
def test_ranks_equal_single_rank(world1, world, tmp_path, cuda):
    parts = _run(world, tmp_path)
    one = world1[0]
    # batched maps: whole maps per rank, contiguous, covering the batch once
    assert [int(p["m0"]) for p in parts] == sorted(int(p["m0"]) for p in parts)
    assert int(parts[0]["m0"]) == 0 and int(parts[-1]["m1"]) == int(one["m1"])
    for a, b in zip(parts, parts[1:]):
        assert int(a["m1"]) == int(b["m0"])
    counts = np.concatenate([p["counts"] for p in parts])
    assert np.array_equal(counts, one["counts"])
    assert np.array_equal(np.concatenate([p["mask_bits"] for p in parts]), one["mask_bits"])
    assert np.concatenate([p["dets"] for p in parts]).tobytes() == one["dets"].tobytes()
    assert all(int(p["total"]) == int(counts.sum()) for p in parts)  # the all-reduced count
    # one large map: owned row slabs cover the rows once, masks and lists equal
    owned = [tuple(int(x) for x in p["owned"]) for p in parts]
    assert owned[0][0] == 0 and owned[-1][1] == int(one["owned"][1])
    for a, b in zip(owned, owned[1:]):
        assert a[1] == b[0]
    assert np.array_equal(np.concatenate([p["big_mask_bits"] for p in parts]), one["big_mask_bits"])
    big = np.concatenate([p["big_dets"] for p in parts])
    ref = one["big_dets"]
    key = lambda d: np.lexsort((d["col"], d["row"]))  # noqa: E731 (lists are sorted per rank)
    assert big[key(big)].tobytes() == ref[key(ref)].tobytes()
    assert all(int(p["big_total"]) == sum(int(q["big_count"]) for q in parts) == int(one["big_count"])
               for p in parts)


def test_bench_gpus2_self_launches_and_counts_match(cuda):
    """bench.py --gpus 2 (no torchrun) re-executes itself under
    torch.distributed.run; the line reports n_gpus 2 and the same detections
    per step as --gpus 1 on the same 256 maps."""
    env = dict(os.environ, UWB_DIST_BACKEND="gloo")
    lines = {}
    for n in (1, 2):
        r = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--steps", "2", "--warmup", "3",
                            "--maps", "256", "--no-e2e", "--no-cpu-baseline"],
                           env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        out = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
        assert len(out) == 1, r.stdout
        lines[n] = out[0]
    assert lines[1]["n_gpus"] == 1 and lines[2]["n_gpus"] == 2
    assert lines[1]["config"]["detections_per_step"] == lines[2]["config"]["detections_per_step"] > 0


def test_bench_refuses_more_gpus_than_visible(cuda):
    import torch
    n = torch.cuda.device_count() + 1
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--steps", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "visible" in r.stdout
