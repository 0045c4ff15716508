"""Build libpsdproj.so in-tree with nvcc for sm_100a (explicit nvcc, no JIT cache)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "psdproj.cu")
DEPS = [os.path.join(HERE, "csrc", f) for f in ("psdproj.cu", "gemm.cuh", "kernels.cuh", "common.cuh", "tridiag.cuh", "cluster_la.cuh", "tridiag_tile.cuh", "gemm_tma.cuh", "tiny_lobpcg.cuh", "sbr.cuh", "tridiag_rep.cuh")] + [
    os.path.join(ROOT, "include", "psdproj.h")]
SO = os.path.join(HERE, "libpsdproj.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-shared",
         "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include")]


def needs_build():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return SO
    cmd = [NVCC] + FLAGS + ["-o", SO + ".tmp", SRC]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
