#!/usr/bin/env bash
# Re-verification after container restore: GPU tests, smoke, bench lines, TB probe.
cd "$(dirname "$0")/.."
O=gpurun_out/r01b
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --config heat --steps 5 --no-cpu > $O/bench_heat.json 2> $O/bench_heat.err
timeout 900 python scripts/tb_probe.py gol int32 8192 100 > $O/tb_gol.txt 2>&1
timeout 900 python scripts/tb_probe.py heat float32 16384 100 > $O/tb_heat.txt 2>&1
ls -la $O
