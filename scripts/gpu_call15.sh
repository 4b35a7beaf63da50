#!/usr/bin/env bash
cd "$(dirname "$0")/.."
O=gpurun_out/c15; mkdir -p $O
timeout 1500 python -m pytest tests/test_multirank_gpu.py -x -q > $O/pytest_multirank.log 2>&1; echo "rc=$?" >> $O/pytest_multirank.log
tail -15 $O/pytest_multirank.log
