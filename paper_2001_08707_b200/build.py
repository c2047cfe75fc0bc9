"""Build libshiftk.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libshiftk.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

def _nccl_dir():
    try:
        import nvidia.nccl
        return list(nvidia.nccl.__path__)[0]
    except Exception:   # headers are needed at build time only; the library is dlopen'ed
        return "/usr"


NCCL_DIR = _nccl_dir()
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                 "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(NCCL_DIR, "include"),
                 "--expt-relaxed-constexpr",
                 '-DSHIFTK_NCCL_DEFAULT="' + os.path.join(NCCL_DIR, "lib", "libnccl.so.2") + '"']
LDFLAGS = ARCH + ["-shared", "-ldl"]
OBJDIR = os.path.join(HERE, "_obj")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "shiftk.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    # one nvcc per translation unit, in parallel (the tiled SpMV instantiations dominate)
    os.makedirs(OBJDIR, exist_ok=True)
    objs, procs = [], []
    for src in sources():
        obj = os.path.join(OBJDIR, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC] + CFLAGS + ["-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd), src))
        objs.append(obj)
    bad = [src for pr, src in procs if pr.wait() != 0]
    if bad:
        raise subprocess.CalledProcessError(1, "nvcc " + " ".join(bad))
    tmp = LIB + ".tmp"
    subprocess.check_call([NVCC] + LDFLAGS + ["-o", tmp] + objs)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
