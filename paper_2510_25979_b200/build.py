"""Builds libattncache.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2510_25979_b200.build [--force] [--verbose-ptxas]

Each csrc/*.cu compiles to build/*.o in parallel, then links into
paper_2510_25979_b200/lib/libattncache.so (static cudart; the CUDA driver API
is reached through cudaGetDriverEntryPoint, so the library has no libcuda
link-time dependency and loads on a GPU-less host).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# ATTNCACHE_BUILD_ROOT / ATTNCACHE_EXTRA_FLAGS: out-of-tree experiment builds (scripts/); the product uses neither
OBJ = os.path.join(os.environ.get("ATTNCACHE_BUILD_ROOT", PKG), "build")
LIB_DIR = os.path.join(os.environ.get("ATTNCACHE_BUILD_ROOT", PKG), "lib")
LIB = os.path.join(LIB_DIR, "libattncache.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC] + os.environ.get("ATTNCACHE_EXTRA_FLAGS", "").split()


def _deps():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "attncache.h")]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _compile(src, obj, ptxas_v):
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    if ptxas_v:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(src)}:\n{r.stdout}\n{r.stderr}")
    return r.stderr


def build(force: bool = False, ptxas_v: bool = False, quiet: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    stamp = os.path.join(OBJ, "flags.txt")  # objects built with other flags are stale
    flags = " ".join(FLAGS)
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        force = True
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = _deps()
    jobs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        if force or _stale(o, [s, *deps]):
            jobs.append((s, o))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for (s, _), log in zip(jobs, ex.map(lambda j: _compile(j[0], j[1], ptxas_v), jobs)):
                if log and not quiet:
                    print(f"--- {os.path.basename(s)}\n{log}", file=sys.stderr)
    objs = [os.path.join(OBJ, os.path.basename(s)[:-3] + ".o") for s in srcs]
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static"])
        os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(flags)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, ptxas_v="--verbose-ptxas" in sys.argv, quiet=False))
