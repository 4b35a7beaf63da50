#!/usr/bin/env bash
cd "$(dirname "$0")/.."
O=gpurun_out/c16; mkdir -p $O
timeout 1500 python -m pytest tests/test_fuzz_paths.py -x -q > $O/pytest_fuzz.log 2>&1; echo "rc=$?" >> $O/pytest_fuzz.log
tail -30 $O/pytest_fuzz.log
