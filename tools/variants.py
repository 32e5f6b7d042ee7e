#!/usr/bin/env python
"""Build A/B variants of libpfresample.so that differ only in -D flags (diagnostics), into
_variants/ (git-ignored): every translation unit is compiled per distinct flag set (objects
cached by a hash of the flags and the sources).  usage:
    python tools/variants.py NAME='-DPF_COPY_CU=4 ...' [NAME2='...' ...]
Then run a tool with PF_LIB_OVERRIDE=_variants/NAME.so."""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1202_6163_b200 import _build  # noqa: E402

OUT = os.path.join(ROOT, "_variants")


def main():
    os.makedirs(OUT, exist_ok=True)
    cflags = [f for f in _build.NVCC_FLAGS if f != "-shared"]
    deps = [os.path.join(_build.CSRC, f) for f in _build.SOURCES + _build.HEADERS]
    stamp = hashlib.sha1(b"".join(open(d, "rb").read() for d in deps)).hexdigest()[:10]
    variants = dict(a.split("=", 1) for a in sys.argv[1:])
    jobs, objs = [], {}
    for name, flags in variants.items():
        key = hashlib.sha1((flags + stamp).encode()).hexdigest()[:10]
        objs[name] = []
        for src in _build.SOURCES:
            o = os.path.join(OUT, f"{src[:-3]}_{key}.o")
            objs[name].append(o)
            if not os.path.exists(o) and o not in [j[-1] for j in jobs]:
                jobs.append([_build._nvcc(), *cflags, *flags.split(), "-c", os.path.join(_build.CSRC, src), "-o", o])
    with ThreadPoolExecutor(max_workers=8) as ex:
        list(ex.map(subprocess.check_call, jobs))
    for name in variants:
        subprocess.check_call([_build._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                               *objs[name], "-o", os.path.join(OUT, f"{name}.so")])
        print(os.path.join(OUT, f"{name}.so"))


if __name__ == "__main__":
    main()
