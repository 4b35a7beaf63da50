#!/usr/bin/env bash
cd "$(dirname "$0")/.."
O=gpurun_out/c26; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_gol.json 2> $O/bench_gol.err; echo "bench rc=$?"
cat $O/bench_gol.json
