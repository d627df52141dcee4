"""Build libreshard_b200.so in-tree: host C++ (g++) + sm_100a CUDA (nvcc), static cudart.

    python -m paper_2312_05181_b200.build [--force]

The library is written next to this file so it travels to the GPU box in the gpurun
snapshot (git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libreshard_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
# /usr/bin/g++ explicitly: the image's CXX=/opt/gcc/bin/g++ wrapper does not link libstdc++.
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _cuda_version() -> str:
    try:
        out = subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout
        line = next(x for x in out.splitlines() if "release" in x)
        return line.split("release")[1].split(",")[0].strip()
    except Exception:
        return "unknown"


def _sources():
    host = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp"))) + [os.path.join(CSRC, "capi.cpp")]
    cuda = sorted(glob.glob(os.path.join(CSRC, "cuda", "*.cu")))
    return host, cuda


def _headers():
    return (glob.glob(os.path.join(CSRC, "**", "*.hpp"), recursive=True)
            + glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
            + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    host, cuda = _sources()
    headers = _headers()
    ver = _cuda_version()
    defs = [f'-DRESHARD_CUDA_VERSION="{ver}"']
    inc = ["-I", CSRC, "-I", os.path.join(CUDA, "include")]
    jobs = []
    for src in host:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        if force or _stale(obj, [src, *headers]):
            jobs.append([CXX, "-std=c++20", "-O2", "-g", "-fPIC", "-Wall", "-Wextra", *defs, *inc, "-c", src, "-o", obj])
    for src in cuda:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        if force or _stale(obj, [src, *headers]):
            jobs.append([NVCC, "-std=c++20", "-O3", "-lineinfo", *ARCH, "-ccbin", CXX, "-Xcompiler", "-fPIC",
                         "-Xptxas", "-v", *defs, *inc, "-c", src, "-o", obj])

    def run(cmd):
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"build failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
        return cmd[-1], p.stderr

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for obj, err in ex.map(run, jobs):
            if verbose and err:
                print(f"[{os.path.basename(obj)}]\n{err}", file=sys.stderr)
    objs = [os.path.join(OBJ, os.path.basename(s) + ".o") for s in host + cuda]
    if force or jobs or _stale(LIB, objs):
        run([NVCC, "-shared", *ARCH, "-ccbin", CXX, "-cudart", "static", "-o", LIB, *objs, "-lpthread"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
