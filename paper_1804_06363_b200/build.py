"""Build librbs.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "librbs.so")
SOURCES = [os.path.join(HERE, "csrc", "api.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in (
    "kernels.cuh", "rbs_internal.cuh", "greedy.inc.cu", "march.cuh", "march2.cuh", "slab.inc.cu")] + [
    os.path.join(ROOT, "include", "rbs.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def nccl_dir() -> str:
    """NCCL of the torch wheel (nvidia-nccl): headers + libnccl.so.2 (mesh slabs over ranks)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for root in (list(spec.submodule_search_locations) if spec else []):
        d = os.path.join(root, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers not found (nvidia-nccl wheel)")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [s for s in SOURCES if os.path.exists(s)]
    deps = [d for d in DEPS if os.path.exists(d)]
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= max(os.path.getmtime(d) for d in deps):
        return SO
    nd = nccl_dir()
    extra = os.environ.get("RBS_NVCC_EXTRA", "").split()   # instrumented builds (tools/)
    cmd = [nvcc()] + NVCC_FLAGS + extra + ["-I" + os.path.join(nd, "include"), "-o", SO] + srcs + [
        "-lcudart", "-L" + os.path.join(nd, "lib"), "-l:libnccl.so.2",
        "-Xlinker", "-rpath," + os.path.join(nd, "lib")]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
