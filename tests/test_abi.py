"""CPU-side checks of the C-ABI boundary (no GPU compute): libpfresample.so loads,
exports every symbol include/pf.h declares, and its host-only helper and
synchronous argument validation behave as documented."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pflib():
    from paper_1202_6163_b200 import _build

    _build.build()
    import paper_1202_6163_b200 as pf

    return pf


def _declared():
    src = open(os.path.join(ROOT, "include", "pf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[A-Za-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(pflib):
    L = pflib.lib()
    declared = _declared()
    assert len(declared) >= 19
    for name in declared:
        assert hasattr(L, name), name
    # the binding covers every declared entry point, with the same names
    assert sorted(pflib.exported_symbols()) == declared


def test_library_is_sm100a(pflib):
    """The built .so carries sm_100a SASS (cuobjdump), not PTX-only or another arch."""
    import shutil
    import subprocess

    cu = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cu):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cu, "--list-elf", pflib.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_required_B_host_helper(pflib, golden_dir):
    """pf_metropolis_required_B (host-only) against the mpmath golden values of Eq. (5)."""
    for line in open(os.path.join(golden_dir, "eq5_required_B.txt")):
        if line.startswith("#") or not line.strip():
            continue
        P, w, e, B = line.split()
        assert pflib.pf_metropolis_required_B(int(P), float(w), float(e)) == int(B)
    assert pflib.pf_metropolis_required_B(0, 0.5, 0.01) == -1
    assert pflib.pf_metropolis_required_B(8, 0.0, 0.01) == -1


def test_argument_validation_is_synchronous(pflib):
    """Invalid arguments return PF_ERR_INVALID_ARG before touching the device (pf.h conventions)."""
    L = pflib.lib()
    dummy = ctypes.c_void_p(16)
    assert L.pf_resample_systematic(None, 10, 1, 0, dummy, None) == 1
    assert L.pf_resample_systematic(dummy, 0, 1, 0, dummy, None) == 1
    assert L.pf_resample_metropolis(dummy, 10, 1, -1, dummy, None) == 1
    assert L.pf_resample_ex(9, dummy, 10, 1, 0, dummy, None, None) == 1
    assert L.pf_resample_batched(3, dummy, 5, 2, 10, 1, 0, 0, dummy, 10, None, None) == 1  # ld < P
    assert L.pf_permute(None, 10, dummy, None) == 1
    assert L.pf_gather_state(dummy, 0, 16, 10, dummy, None) == 1
    assert L.pf_status_string(1) == b"PF_ERR_INVALID_ARG"
    assert pflib.pf_workspace_bytes("systematic", 1024, 65536) > 1024 * 65536 * 8


def test_no_cpu_fallback(pflib):
    """The product path refuses CPU tensors (no silent fallback)."""
    import torch

    with pytest.raises(pflib.PfError):
        pflib.pf_resample_systematic(torch.zeros(8), 1)


def test_product_path_does_not_import_oracle():
    """Neither the binding nor the CUDA sources reference oracle/ (independence)."""
    pkg = os.path.join(ROOT, "paper_1202_6163_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "pfo_" not in txt, f
                assert "pfo.h" not in txt
