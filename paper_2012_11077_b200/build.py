"""Build recipe for the native libraries (sm_100a only).

* ``lib/libuwbvital_b200.so`` - CUDA kernels + the C ABI (include/uwbvital_b200.h)
* ``lib/libuwbvital.so``      - the C++ drop-in (include/uwbvital/*.hpp) over the C ABI

Both are built in-tree so they travel to the GPU box with the repository
snapshot. nvcc cross-compiles without a GPU.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
INCLUDE = os.path.join(ROOT, "include")

CUDA_SOURCES = ["sat.cu", "sat_cluster.cu", "cfar.cu", "cfar_ring.cu", "cfar_fused.cu", "cfar_cert.cu", "frontend.cu", "ingest.cu", "capi.cu"]
HEADERS = ["common.cuh", "kernels.cuh", "cfar_common.cuh"]
NVCC = os.environ.get("NVCC", "nvcc")
CXX = os.environ.get("CXX", "g++")

# --fmad=false and -ffp-contract=off: the reference is evaluated without FMA
# contraction; the kernels reproduce its rounding bit for bit.
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-I" + INCLUDE,
]

# tuning build for the scripts/ probes only: environment knobs (common.cuh UWB_KNOB)
if os.environ.get("UWB_TUNING_KNOBS") == "1":
    NVCC_FLAGS.append("-DUWB_TUNING_KNOBS")
# device-side bounds checks (the compute-sanitizer stand-in)
if os.environ.get("UWB_DEVICE_CHECKS") == "1":
    NVCC_FLAGS.append("-DUWB_DEVICE_CHECKS")

CAPI_SO = os.path.join(LIB, "libuwbvital_b200.so")
DROPIN_SO = os.path.join(LIB, "libuwbvital.so")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str], verbose: bool):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose: bool = False, force: bool = False) -> None:
    os.makedirs(LIB, exist_ok=True)
    cu = [os.path.join(CSRC, s) for s in CUDA_SOURCES]
    deps = cu + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "uwbvital_b200.h")]
    if force or _stale(CAPI_SO, deps):
        objs = []
        for src in cu:
            obj = os.path.join(LIB, os.path.basename(src) + ".o")
            if force or _stale(obj, [src] + deps[len(cu):]):
                _run([NVCC, *NVCC_FLAGS, "-c", src, "-o", obj], verbose)
            objs.append(obj)
        _run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", CAPI_SO],
             verbose)
    dropin_src = os.path.join(CSRC, "dropin.cpp")
    hdrs = [os.path.join(INCLUDE, "uwbvital", h) for h in os.listdir(os.path.join(INCLUDE, "uwbvital"))]
    if force or _stale(DROPIN_SO, [dropin_src, CAPI_SO, *hdrs]):
        _run([CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-I" + INCLUDE,
              dropin_src, "-L" + LIB, "-luwbvital_b200", "-Wl,-rpath,$ORIGIN", "-o", DROPIN_SO],
             verbose)


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
