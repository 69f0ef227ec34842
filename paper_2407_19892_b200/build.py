"""Build libggm.so in-tree with nvcc for sm_100a (no JIT cache, so the .so travels with the
repository snapshot to the GPU box).  Usage: ``python -m paper_2407_19892_b200.build``."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build_obj")
LIB = os.path.join(PKG, "libggm.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "-Xptxas", "-warn-spills"]

SOURCES = ["ggm_api.cu", "sparse_precision.cu", "grid_solve.cu", "gram_eig.cu", "gram_tc.cu", "wald.cu"]
HEADERS = ["ggm_internal.h", "ptx_sm100.cuh"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def _needs(obj, src):
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(PKG, "..", "include", "ggm.h"), os.path.abspath(__file__)]
    return _mtime(obj) < max(_mtime(d) for d in deps)


def _compile(src):
    s = os.path.join(CSRC, src)
    o = os.path.join(OBJ, src.replace(".cu", ".o"))
    if not _needs(o, s):
        return o, ""
    cmd = [NVCC, *ARCH, *FLAGS, "-c", s, "-o", o]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return o, r.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(_compile, SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log.strip():
                print(log)
    if _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcublas", "-lcusolver", "-lcusparse",
               f"-L{CUDA_HOME}/lib64", "-Xlinker", f"-rpath,{CUDA_HOME}/lib64"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
