"""The C++ host API (include/wgtb/stencil.hpp) and user customising functions
(include/wgtb/stencil_custom.cuh) on the GPU: tests/cpp/api_test.cu, built
into paper_1511_02490_b200/lib/api_test, checks a user functor with an
asymmetric border region against direct host loops for both load paths,
several K and block shapes, plus the built-in GoL through Stencil<int32_t>."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent.parent / "paper_1511_02490_b200" / "lib" / "api_test"


@pytest.mark.gpu
def test_cpp_api_and_custom_functor():
    assert BIN.exists(), "run __graft_entry__.build() first"
    proc = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0 and proc.stdout.strip().endswith("OK"), proc.stdout + proc.stderr


def test_cpp_api_binary_built():
    assert BIN.exists()
