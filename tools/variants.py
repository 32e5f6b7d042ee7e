#!/usr/bin/env python
"""Build A/B variants of libpfresample.so that differ only in pf_fused.cu's -D flags
(diagnostics; the other translation units are compiled once and shared), into _variants/
(git-ignored).  usage: python tools/variants.py NAME='-DPF_COPY_CU=4 ...' [NAME2='...' ...]
Then run a tool with PF_LIB_OVERRIDE=_variants/NAME.so."""
from __future__ import annotations

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
    others = [s for s in _build.SOURCES if s != "pf_fused.cu"]
    objs = {s: os.path.join(OUT, s.replace(".cu", ".o")) for s in others}
    jobs = []
    for s, o in objs.items():
        src = os.path.join(_build.CSRC, s)
        if not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(src), *[
                os.path.getmtime(os.path.join(_build.CSRC, h)) for h in _build.HEADERS]):
            jobs.append([_build._nvcc(), *cflags, "-c", src, "-o", o])
    variants = dict(a.split("=", 1) for a in sys.argv[1:])
    for name, flags in variants.items():
        jobs.append([_build._nvcc(), *cflags, *flags.split(), "-c", os.path.join(_build.CSRC, "pf_fused.cu"),
                     "-o", os.path.join(OUT, f"fused_{name}.o")])
    with ThreadPoolExecutor(max_workers=8) as ex:
        list(ex.map(subprocess.check_call, jobs))
    for name in variants:
        subprocess.check_call([_build._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                               os.path.join(OUT, f"fused_{name}.o"), *objs.values(), "-o",
                               os.path.join(OUT, f"{name}.so")])
        print(os.path.join(OUT, f"{name}.so"))


if __name__ == "__main__":
    main()
