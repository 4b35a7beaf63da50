#!/usr/bin/env bash
# One GPU call: full gpu test suite, default bench line, bit-plane probe.
cd "$(dirname "$0")/.."
O=gpurun_out/check; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
cat $O/bench.json
timeout 900 python scripts/bits_probe.py > $O/bits_probe.txt 2>&1
head -8 $O/bits_probe.txt
