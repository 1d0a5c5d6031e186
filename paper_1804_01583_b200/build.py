"""Build libkrylov_reach.so in-tree with nvcc for sm_100a (B200).

Links NCCL from the torch wheel (site-packages/nvidia/nccl) so the process holds one NCCL — the same
one torch.distributed loads. cudart is linked statically. Usage: python -m paper_1804_01583_b200.build
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libkrylov_reach.so")
SRCS = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
HDRS = sorted(glob.glob(os.path.join(HERE, "csrc", "*.h"))) + [os.path.join(ROOT, "include", "krylov_reach.h")]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SRCS + HDRS)


def build(force=False, verbose=False, out=None):
    """Compile each translation unit in parallel (nvcc -c), then link the shared library. out: another
    output path (A/B builds of kernel variants under scratch_libs/); the product loads only LIB."""
    out = out or LIB
    if out == LIB and not force and not needs_build():
        return LIB
    inc, lib = nccl_dirs()
    flags = [nvcc(), "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
             "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
             "-I", os.path.join(ROOT, "include"), "-I", inc] + os.environ.get("KR_NVCC_FLAGS", "").split()
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in SRCS]
    from concurrent.futures import ThreadPoolExecutor

    def one(so):
        src, obj = so
        return subprocess.run(flags + ["-c", "-o", obj, src], capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=min(len(SRCS), os.cpu_count() or 4)) as ex:
        results = list(ex.map(one, zip(SRCS, objs)))
    for r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libkrylov_reach.so")
        if verbose:
            sys.stderr.write(r.stderr)
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out] + objs + \
          ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libkrylov_reach.so")
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
