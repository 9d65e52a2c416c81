"""Build libsimdx.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build()."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsimdx.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-O2", "-shared", "-diag-suppress", "177,550"]


def nccl_dir() -> str:
    """NCCL 2.28 shipped with the torch wheel (nvidia-nccl-cu12): headers + libnccl.so.2."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl.h not found (expected the nvidia-nccl wheel next to torch)")


def link_flags():
    d = nccl_dir()
    lib = os.path.join(d, "lib")
    return ["-I", os.path.join(d, "include"), "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(os.path.dirname(HERE), "include", "simdx.h")]


def _compile_all(out: str, extra: list) -> None:
    """One nvcc per translation unit, in parallel (the .cu files are independent:
    no relocatable device code), then one link into the shared library."""
    from concurrent.futures import ThreadPoolExecutor
    objdir = out + ".objs"
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"]
    inc = [f for f in link_flags() if f.startswith("-I")] + [link_flags()[1]]

    def one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        subprocess.check_call([NVCC, *cflags, *extra, "-c", "-o", obj, src, *inc])
        return obj

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(one, sources()))
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                           "-o", out + ".tmp", *objs, *link_flags()])
    os.replace(out + ".tmp", out)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in deps()):
            return LIB
    _compile_all(LIB, ["-Xptxas", "-v"] if verbose else [])
    return LIB


def build_variant(name: str, defines: list) -> str:
    """An experiment build (profiles/: loaded with SIMDX_LIB=...), e.g. -DSX_PROBE=8."""
    out = os.path.join(os.path.dirname(HERE), "build", f"libsimdx_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    _compile_all(out, list(defines))
    return out


if __name__ == "__main__":
    import sys
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:]))
    else:
        build(force=True, verbose="-v" in sys.argv)
        print(LIB)
