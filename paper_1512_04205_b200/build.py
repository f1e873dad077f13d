"""Build libcdmd.so in-tree with nvcc for sm_100a (no torch types, plain C ABI).

    python -m paper_1512_04205_b200.build        # or build() from __graft_entry__
"""

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libcdmd.so")
SOURCES = ["api.cu", "sensing.cu", "sketch.cu", "fit.cu", "modes.cu", "modes_tc.cu", "foreground.cu", "foreground_tc.cu", "eig.cu", "eigh.cu", "sketch_tc.cu", "sketch_tc2.cu", "median3.cu", "partition.cu", "amplitudes.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def cuda_home():
    return os.path.dirname(os.path.dirname(nvcc()))


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "cdmd.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=True):
    if not force and not _stale():
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    cuda = cuda_home()
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
           "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES],
           "-L", os.path.join(cuda, "lib64"), "-lcusolver", "-lcublas",
           "-Xlinker", "-rpath=" + os.path.join(cuda, "lib64"),
           *os.environ.get("CDMD_EXTRA_NVCC", "").split()]   # e.g. -DCDMD_GS_PROF (instrumented builds)
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
