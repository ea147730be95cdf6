"""Build libbbc.so in-tree with nvcc for sm_100a (the C-ABI library of include/bbc.h)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
# BBC_LIB_OUT / BBC_NVCC_DEFS: build a variant library elsewhere with extra -D flags (kernel
# tuning experiments; the default build and the product path ignore them)
LIB = os.environ.get("BBC_LIB_OUT") or os.path.join(HERE, "libbbc.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("bbc_api.cu",)]
# every header the library includes: an edit to any of them rebuilds it (stale())
DEPS = SOURCES + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [
    os.path.join(ROOT, "include", "bbc.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir() -> str:
    """NCCL shipped with PyTorch's nvidia-nccl wheel (the library torch itself loads)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        return list(spec.submodule_search_locations)[0]
    return "/usr"
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        nccl = _nccl_dir()
        defs = os.environ.get("BBC_NVCC_DEFS", "").split()
        cmd = [NVCC, *FLAGS, *defs, "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include"),
               *SOURCES, "-o", LIB + ".tmp", "-lcudart", "-L", os.path.join(nccl, "lib"),
               "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libbbc.so")
        if verbose:
            sys.stderr.write(r.stderr)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
