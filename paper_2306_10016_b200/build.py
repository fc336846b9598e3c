"""Build libhdconv.so in-tree for sm_100a (nvcc; no GPU needed to compile).

    python -m paper_2306_10016_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libhdconv.so")
BUILD = os.path.join(HERE, "csrc", "build")
SOURCES = ["hd_kernels.cu", "hd_api.cu", "hd_dist.cu", "hd_filter.cu", "hd_k_s512.cu", "hd_k_s2048r.cu", "hd_k_s4096r.cu", "hd_k_s128.cu"] + [f"hd_k_{d}_{n}.cu" for d in ("f64", "f32") for n in (256, 576, 1024)]
HEADERS = ["hd_device.cuh", "hd_internal.h", "hd_kernels.cuh", "hd_w512.cuh", "hd_s512.cuh", "hd_s2048r.cuh", "hd_s4096r.cuh", "hd_w256.cuh", "hd_s128.cuh", "hd_s512c.cuh", "hd_tma.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-I" + INCLUDE, "-I" + CSRC]


def _newest_input() -> float:
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(INCLUDE, "hdconv.h"),
                                                                 os.path.abspath(__file__)]
    for src in SOURCES:  # every header a source includes, listed or not
        files += sorted(_deps(os.path.join(CSRC, src)))
    return max(os.path.getmtime(f) for f in files)


def _deps(path: str, seen: set | None = None) -> set:
    """Transitive local #include "..." dependencies of a source file."""
    seen = set() if seen is None else seen
    for line in open(path):
        line = line.strip()
        if line.startswith("#include \""):
            name = line.split("\"")[1]
            for d in (CSRC, INCLUDE):
                f = os.path.join(d, name)
                if os.path.exists(f) and f not in seen:
                    seen.add(f)
                    _deps(f, seen)
    return seen


def _compile(src: str) -> str:
    obj = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
    path = os.path.join(CSRC, src)
    newest = max(os.path.getmtime(f) for f in _deps(path) | {path, os.path.abspath(__file__)})
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj
    cmd = [NVCC] + FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_input():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp] + objs + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
