"""NS-4 on the device: the folded dexp() / weight2() of pf_device.cuh against the literal NS-4
transcription for every float32 t <= 0 (2^31 + 1 inputs, NaNs included), bit for bit.  The
folding (clamp for step 1, no step 2, add-and-subtract rint for step 3) is argued in
pf_device.cuh; this is the exhaustive check (tools/dexp_check.cu), built here for sm_100a."""
from __future__ import annotations

import json
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_dexp_folded_steps_bit_identical_exhaustive(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = tmp_path / "dexp_check"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-I",
                    os.path.join(ROOT, "paper_1202_6163_b200", "csrc"), os.path.join(ROOT, "tools", "dexp_check.cu"),
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["cuda"] == "no error"
    assert res["inputs"] == (1 << 31) + 1
    assert res["mismatches"] == 0, out.stdout
