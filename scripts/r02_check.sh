#!/usr/bin/env bash
# Round-2 quick GPU check: selected GPU tests + the full bench line.
cd "$(dirname "$0")/.."
O=gpurun_out/r02b; mkdir -p $O
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt
timeout 900 python -m pytest tests/test_baseline_configs.py -m gpu -q -x > $O/pytest_cfg.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest_cfg.log
tail -3 $O/pytest_cfg.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -c 3000 $O/bench.err
timeout 600 python bench.py --impl reference --steps 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
cat $O/bench_ref.json
