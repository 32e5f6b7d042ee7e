"""Build libpfresample.so in-tree with nvcc for sm_100a (no JIT cache)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpfresample.so")
SOURCES = ["pf_kernels.cu", "pf_fused.cu", "pf_migrate.cu", "pf_f64.cu", "pf_wsort.cu", "pf_api.cu"]
HEADERS = ["pf_device.cuh", "pf_internal.h"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    # keep IEEE float semantics (no fast-math, no FTZ): the float -> integer
    # boundary must be bit-identical to the oracle (DESIGN.md §3 NS-4)
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=false",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(PKG), "include", "pf.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    """Each translation unit compiles in its own nvcc process (in parallel), then one link."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    tag = f".tmp{os.getpid()}"
    objs = [os.path.join(PKG, f"_{os.path.splitext(s)[0]}{tag}.o") for s in SOURCES]
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]
    cmds = [[_nvcc(), *cflags, "-c", os.path.join(CSRC, s), "-o", o] for s, o in zip(SOURCES, objs)]
    try:
        with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
            for cmd in cmds:
                if verbose:
                    print(" ".join(cmd))
            list(ex.map(subprocess.check_call, cmds))
        tmp = LIB + tag
        link = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", tmp]
        if verbose:
            print(" ".join(link))
        subprocess.check_call(link)
        os.replace(tmp, LIB)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
