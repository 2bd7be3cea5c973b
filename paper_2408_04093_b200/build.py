"""In-tree build of libtreedec_b200.so (sm_100a) with nvcc.

The shared library is written next to this file so that it travels to the GPU
box with the repo snapshot (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtreedec_b200.so")
SOURCES = ["td_kernels.cu", "td_capi.cu", "td_nccl_dev.cu"]
HEADERS = ["td_device.cuh", "td_internal.h"]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "--expt-relaxed-constexpr",
    "-I" + os.path.join(ROOT, "include"),
]


def _nccl_device_include() -> str | None:
    """NCCL's device-API headers (NCCL >= 2.28, shipped with torch's NCCL wheel)."""
    cands = [os.environ.get("TD_NCCL_INCLUDE")]
    try:
        import nvidia.nccl
        cands += [os.path.join(p, "include") for p in nvidia.nccl.__path__]
    except ImportError:
        pass
    for c in cands:
        if c and os.path.exists(os.path.join(c, "nccl_device.h")):
            return c
    return None


def _extra_flags(src: str) -> list[str]:
    if src != "td_nccl_dev.cu":
        return []
    inc = _nccl_device_include()
    return ["-I" + inc, "-DTD_HAVE_NCCL_DEVICE"] if inc else []


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "treedec_b200.h"))
    deps.append(__file__)
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every CUDA source for sm_100a and link libtreedec_b200.so."""
    if not force and not _stale():
        return LIB
    objs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [_nvcc(), *NVCC_FLAGS, *_extra_flags(src), "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp, "-ldl"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
