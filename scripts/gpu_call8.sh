#!/usr/bin/env bash
cd "$(dirname "$0")/.."
O=gpurun_out/c8; mkdir -p $O
timeout 600 python -m pytest tests/test_peer_halo.py tests/test_cross_strips.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -5 $O/pytest.log
