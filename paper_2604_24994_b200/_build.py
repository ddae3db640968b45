"""Builds libpowerfoam.so (the C-ABI library, include/powerfoam.h) in-tree with nvcc
for sm_100a.  Called by __graft_entry__.build() and, lazily, by the binding."""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libpowerfoam.so")
SOURCES = ["pf_api.cu", "pf_prep.cu", "pf_sort.cu", "pf_raster.cu", "pf_cech.cu", "pf_trace.cu"]
HEADERS = ["pf_internal.cuh", "pf_pixel.cuh", "pf_bvh.cuh", os.path.join("..", "..", "include", "powerfoam.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found: cannot build libpowerfoam.so")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile libpowerfoam.so; `out`/`defines` build an A/B variant elsewhere
    (selected at run time with PF_LIBRARY_PATH)."""
    target = os.path.abspath(out) if out else LIB
    if out is None and not force and not _stale():
        return LIB
    tmp = target + f".tmp{os.getpid()}"
    cmd = [nvcc(), "-std=c++17", "-O3", "-lineinfo", *ARCH, "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(ROOT, "include"),
           *[f"-D{d}" for d in defines], "-o", tmp] + [os.path.join(CSRC, f) for f in SOURCES]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force=True, verbose=True))
