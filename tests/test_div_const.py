"""The fp32 division by the boxmean cell count 28 (ops.cuh div_const_rn<28>,
used by the config-4 kernel) is bit-identical to IEEE division for every one
of the 2^32 inputs: an exhaustive GPU check (tests/cuda/div_const_check.cu,
built with the library's own flags)."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_div_const_28_exhaustive(tmp_path):
    exe = tmp_path / "div_const_check"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "-fmad=false", "-I", str(ROOT / "paper_1511_02490_b200" / "csrc" / "stencil"),
                    str(ROOT / "tests" / "cuda" / "div_const_check.cu"), "-o", str(exe)], check=True,
                   timeout=300)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and " 0 mismatches" in out.stdout, out.stdout + out.stderr
