"""Build libdtwlb.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_0811_3301_b200.build [--force]

Objects are compiled in parallel and linked into ``paper_0811_3301_b200/libdtwlb.so``
(git-ignored, but shipped to the GPU box by gpurun).  The CUDA runtime is linked
statically so the library does not depend on which libcudart torch loaded.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
CHECKED = os.environ.get("DTWLB_CHECKED") == "1"  # debug build with device bounds checks
LIB = os.path.join(HERE, "libdtwlb_checked.so" if CHECKED else "libdtwlb.so")
OBJ = os.path.join(HERE, "_obj_checked" if CHECKED else "_obj")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
SOURCES = ["abi.cu", "envelope.cu", "keogh.cu", "stream.cu", "improved.cu", "dtw.cu", "dtw_wide.cu", "search.cu",
           "comm.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-I", INCLUDE] + (["-DDTWLB_CHECKED"] if CHECKED else [])


def _deps_mtime() -> float:
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "dtwlb.h")]
    return max(os.path.getmtime(f) for f in files)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(OBJ, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + f".{os.getpid()}.tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           "-o", tmp, *objs, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
