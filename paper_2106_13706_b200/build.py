"""Build libddks.so in-tree for sm_100a (nvcc, explicit -gencode; no JIT cache, no torch extension).

NCCL: compiled and linked against the NCCL that torch bundles (site-packages/nvidia/nccl, 2.28.x), NOT the
system 2.27 in /usr/include — both use soname libnccl.so.2 and only one can be live in a torch process.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libddks.so")
SOURCES = [os.path.join(HERE, "csrc", "ddks_api.cu")]
DEPS = SOURCES + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "ddks.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    for p in sys.path:
        cand = os.path.join(p, "nvidia", "nccl")
        if os.path.exists(os.path.join(cand, "include", "nccl.h")):
            return cand
    raise RuntimeError("torch-bundled NCCL (site-packages/nvidia/nccl) not found")


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return SO
    nd = nccl_dir()
    tmp = SO + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-fvisibility=hidden",
           "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(nd, "include"), "-I", os.path.join(ROOT, "include"),
           "-o", tmp, *SOURCES,
           "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", f"-Xlinker=-rpath={os.path.join(nd, 'lib')}",
           "-lcudart"]
    subprocess.check_call(cmd)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
