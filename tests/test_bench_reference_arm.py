"""bench.py's reference arm runs on the host alone (no GPU): one JSON line
with the driver's keys, impl=reference, the same `config` object as our arm,
and a cpu_baseline / e2e that describe the same run.  It must
never load the product library: its inputs come from oracle_fill."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

RUNNER = """
import runpy, sys
sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '3']
runpy.run_path('bench.py', run_name='__main__')
maps = open('/proc/self/maps').read()
print('LOADED_SK', 'libsk_stencil' in maps, 'LOADED_WGTB', 'libwgtb' in maps)
"""


def test_reference_arm_json_line():
    proc = subprocess.run([sys.executable, "-c", RUNNER], cwd=ROOT, capture_output=True,
                          text=True, timeout=900)
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert proc.returncode == 0 and len(lines) == 1, proc.stdout + proc.stderr[-2000:]
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "Gcells/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["warmup"] >= 3
    # same workload object as our arm prints
    sys.path.insert(0, str(ROOT))
    import bench

    assert d["config"] == bench.workload_config("gol", 1, "weak")
    assert "LOADED_SK False LOADED_WGTB False" in proc.stdout, proc.stdout[-500:]


def test_bench_gpus_flag_relaunches_under_torchrun(monkeypatch):
    """--gpus N outside torchrun re-executes under torch.distributed.run with
    N ranks (the driver may call `python bench.py --gpus 8`)."""
    sys.path.insert(0, str(ROOT))
    import bench

    calls = []
    monkeypatch.setattr(subprocess, "call", lambda cmd: calls.append(cmd) or 0)

    class A:
        gpus = 4

    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    assert bench.relaunch_distributed(A()) == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "2"]
