"""The histogram-cell shortcut of the NEXT-1 kernel (paper_2604_13191_b200/csrc/hist_cells.cuh:
cells from rsqrt.approx unless a component is within 1e-5 of a cell boundary) returns the
pinned cell (PREDICATES §10) whenever it decides one: 1.5e8 random and boundary-neighbourhood
inputs on the device, compiled with the library's flags."""
import os
import subprocess

import pytest

from paper_2604_13191_b200 import build as vb

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.gpu
def test_hist_cell_fast_equals_pinned(tmp_path):
    exe = str(tmp_path / "hist_cells_check")
    flags = [f for f in vb.NVCC_FLAGS if f not in ("-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-Xptxas", "-v")]
    subprocess.run([vb.NVCC] + flags + [os.path.join(HERE, "cuda", "hist_cells_check.cu"), "-o", exe],
                   check=True, capture_output=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("mismatches 0 ")
