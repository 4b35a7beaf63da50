"""Multi-rank paths on the GPU: (1) row-sharded iteration on the CUDA
executor with halo exchange (2 and 3 ranks) is bit-identical to the oracle;
(2) the bench.py --gpus 2 launch (torchrun, barrier, max-over-ranks timing,
one JSON line on rank 0) works end to end.  Ranks share the single GPU of a
gpurun box through the gloo backend."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def torchrun(n, *args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n), *args]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)


@pytest.mark.parametrize("n", [2, 3])
def test_sharded_cuda_iteration_matches_oracle(n):
    proc = torchrun(n, str(ROOT / "tests" / "mp_gpu_worker.py"))
    assert "ALL_OK" in proc.stdout, proc.stdout + proc.stderr[-3000:]


@pytest.mark.parametrize("transport", ["peer", "nccl"])
def test_bench_two_ranks_json_line(transport):
    """transport=peer: IPC-mapped peer stores from the strip kernel;
    transport=nccl: the send/recv schedule (host-staged under gloo here)."""
    proc = torchrun(2, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "3", "--wc", "32",
                    "--wr", "8", "--no-cpu", "--backend", "gloo", "--transport", transport)
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert proc.returncode == 0 and len(lines) == 1, proc.stdout + proc.stderr[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["global_grid"] == "8192x16384"
    assert d["e2e"]["value"] > 0
    assert (d["transport"] == "peer") == (transport == "peer")


def test_bench_two_ranks_heat_temporal_leg():
    """Config 3 at N=2 (ranks sharing the GPU): the headline peer schedule and
    the temporally blocked peer schedule (TB-deep halos) agree bit for bit."""
    proc = torchrun(2, "bench.py", "--gpus", "2", "--config", "heat", "--steps", "1", "--warmup", "3",
                    "--wc", "104", "--wr", "6", "--no-cpu", "--no-e2e", "--backend", "gloo", timeout=900)
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert proc.returncode == 0 and len(lines) == 1, proc.stdout + proc.stderr[-3000:]
    d = json.loads(lines[0])
    assert d["transport"] == "peer"
    t = d["temporal_blocking"]
    assert t and t["bit_exact_vs_one_pass"] and t["value"] > 0


def test_bench_two_ranks_strong_scaling():
    """--scaling strong splits the configured grid across the ranks."""
    proc = torchrun(2, "bench.py", "--gpus", "2", "--scaling", "strong", "--steps", "1", "--warmup", "3",
                    "--wc", "32", "--wr", "8", "--no-cpu", "--no-e2e", "--backend", "gloo")
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert proc.returncode == 0 and len(lines) == 1, proc.stdout + proc.stderr[-3000:]
    d = json.loads(lines[0])
    assert d["scaling"] == "strong" and d["config"]["global_grid"] == "8192x8192"
    assert "8192x4096 per GPU" in d["config"]["workload"]
