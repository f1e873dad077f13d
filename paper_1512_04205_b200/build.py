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
SOURCES = ["api.cu", "sensing.cu", "sketch.cu", "fit.cu", "modes.cu", "modes_tc.cu", "foreground.cu", "foreground_tc.cu", "eig.cu", "eigh.cu", "sketch_tc.cu", "sketch_tc2.cu", "median3.cu", "partition.cu", "amplitudes.cu", "fused_tc.cu", "sparse_csc.cu", "lanczos.cu"]
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
    stamp = os.path.join(HERE, "lib", "obj", "flags")   # the library was built with other extra flags
    if (open(stamp).read() if os.path.exists(stamp) else "") != os.environ.get("CDMD_EXTRA_NVCC", ""):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "cdmd.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, obj, cuda, verbose):
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-c", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
           "-I", os.path.join(ROOT, "include"), "-o", obj + ".tmp", src,
           *os.environ.get("CDMD_EXTRA_NVCC", "").split()]   # e.g. -DCDMD_ABLATIONS (instrumented builds)
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(obj + ".tmp", obj)


def build(force=False, verbose=True):
    """Compile every source to an object (in parallel; an object is rebuilt when its
    source, a header or this file is newer), then link libcdmd.so."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "lib", "obj")
    os.makedirs(objdir, exist_ok=True)
    cuda = cuda_home()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith(".cu")]
    headers += [os.path.join(ROOT, "include", "cdmd.h"), __file__]
    hdr_t = max(os.path.getmtime(h) for h in headers)
    extra = os.environ.get("CDMD_EXTRA_NVCC", "")
    stamp = os.path.join(objdir, "flags")
    flags_changed = not os.path.exists(stamp) or open(stamp).read() != extra
    jobs = []
    for s in SOURCES:
        src, obj = os.path.join(CSRC, s), os.path.join(objdir, s + ".o")
        if force or flags_changed or not os.path.exists(obj) or \
                os.path.getmtime(obj) < max(os.path.getmtime(src), hdr_t):
            jobs.append((src, obj))
    with ThreadPoolExecutor(max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for f in [ex.submit(_compile, a, b, cuda, verbose) for a, b in jobs]:
            f.result()
    with open(stamp, "w") as fh:
        fh.write(extra)
    cmd = [nvcc(), *ARCH, "-shared", "-o", LIB + ".tmp", *[os.path.join(objdir, s + ".o") for s in SOURCES],
           "-L", os.path.join(cuda, "lib64"), "-lcusolver", "-lcublas",
           "-Xlinker", "-rpath=" + os.path.join(cuda, "lib64")]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
