"""The C-ABI NCCL halo schedule (sk_stencil_iterate_nccl, csrc/stencil/
nccl_halo.cu; SURVEY.md §8b "sk_halo_step(..., ncclComm_t)", §8e):

* tests/cpp/nccl_halo_test.cu runs 1-8 thread-ranks on one GPU over an NCCL
  test double (tests/cpp/fake_nccl.cpp, soname libnccl.so.2 - real NCCL
  refuses two ranks on one device) and requires the gathered result to equal
  the single-GPU iterate bit for bit;
* a real NCCL communicator (torch's) drives it at world 1 here, and at world
  2 under torchrun with the NCCL backend when the box has >= 2 GPUs."""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "paper_1511_02490_b200" / "lib" / "nccl_halo_test"
WORKER = ROOT / "tests" / "nccl_abi_worker.py"


def test_nccl_halo_test_built():
    assert BIN.exists(), "run __graft_entry__.build() first"


@pytest.mark.gpu
def test_nccl_schedule_thread_ranks_on_one_gpu():
    proc = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0 and proc.stdout.strip().endswith("OK"), proc.stdout + proc.stderr


def _torchrun(n: int, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29650 + n), str(WORKER)]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)


@pytest.mark.gpu
def test_nccl_abi_world1_real_nccl():
    proc = _torchrun(1)
    assert "ALL_OK" in proc.stdout, proc.stdout + proc.stderr[-3000:]


@pytest.mark.gpu
def test_nccl_abi_world2_real_nccl():
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs: NCCL does not run two ranks on one device")
    proc = _torchrun(2)
    assert "ALL_OK" in proc.stdout, proc.stdout + proc.stderr[-3000:]
