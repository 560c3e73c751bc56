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
SOURCES = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))  # one translation unit per C-ABI area
DEPS = SOURCES + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + glob.glob(os.path.join(HERE, "csrc", "*.h")) + \
    [os.path.join(ROOT, "include", "ddks.h")]
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
    debug = ["-DDDKS_DEBUG"] if os.environ.get("DDKS_DEBUG") else []  # device-side bounds asserts (ddks_common.cuh)
    debug += os.environ.get("DDKS_NVCC_EXTRA", "").split()  # experiments only (e.g. -DDDKS_CFG5=8,384,256,3)
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", *debug, "-Xcompiler", "-fPIC,-fvisibility=hidden",
              "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(nd, "include"), "-I", os.path.join(ROOT, "include")]
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    tmp = SO + f".tmp{os.getpid()}"
    try:
        for src in SOURCES:  # the translation units compile in parallel
            obj = os.path.join(objdir, os.path.basename(src)[:-3] + f".{os.getpid()}.o")
            objs.append(obj)
            procs.append(subprocess.Popen(common + ["-c", src, "-o", obj]))
        rcs = [p.wait() for p in procs]
        if any(rcs):
            raise subprocess.CalledProcessError(max(rcs), "nvcc -c")
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L", os.path.join(nd, "lib"),
                               "-l:libnccl.so.2", f"-Xlinker=-rpath={os.path.join(nd, 'lib')}", "-lcudart"])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
