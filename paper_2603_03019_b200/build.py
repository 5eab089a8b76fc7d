"""Build libhq.so (the C-ABI library) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import concurrent.futures
import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libhq.so")
SOURCES = [os.path.join(PKG, "csrc", n) for n in ("hq_api.cu", "hq_kernels.cu", "hq_v2.cu", "hq_v3.cu", "hq_batch.cu")]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    "-I", os.path.join(ROOT, "include"),
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = SOURCES + glob.glob(os.path.join(PKG, "csrc", "*.h")) + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + \
        [os.path.join(ROOT, "include", "hq.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile libhq.so (or a variant at `out` with extra -D defines, for A/B runs)."""
    lib = out or LIB
    if force or out or _stale():
        nvcc = os.environ.get("NVCC", "nvcc")
        extra = ["-DHQ_DEBUG_HANG"] if os.environ.get("HQ_DEBUG_HANG") else []
        extra += ["-D" + d for d in defines]
        extra += os.environ.get("HQ_NVCC_EXTRA", "").split()   # development: extra nvcc flags
        # one object per translation unit, compiled in parallel, then one shared-library link
        flags = [f for f in NVCC_FLAGS if f != "-shared"] + extra + (["-Xptxas", "-v"] if verbose else [])
        objdir = os.path.join(PKG, "build", os.path.basename(lib) + ".o")
        os.makedirs(objdir, exist_ok=True)
        objs = [os.path.join(objdir, os.path.basename(src)[:-3] + ".o") for src in SOURCES]
        with concurrent.futures.ThreadPoolExecutor(len(SOURCES)) as ex:
            futs = [ex.submit(subprocess.run, [nvcc] + flags + ["-c", "-o", o, src], check=True)
                    for src, o in zip(SOURCES, objs)]
            for f in futs:
                f.result()
        subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib] + objs, check=True)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
