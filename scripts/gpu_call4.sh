#!/usr/bin/env bash
# Strip kernel + peer exchange: parity tests, heat strip probe, multirank bench tests.
cd "$(dirname "$0")/.."
O=gpurun_out/c4; mkdir -p $O
timeout 900 python -m pytest tests/test_cross_strips.py -x -q > $O/pytest_strips.log 2>&1; echo "rc=$?" >> $O/pytest_strips.log
tail -3 $O/pytest_strips.log
timeout 600 python -m pytest tests/test_peer_halo.py -x -q > $O/pytest_peer.log 2>&1; echo "rc=$?" >> $O/pytest_peer.log
tail -3 $O/pytest_peer.log
timeout 900 python scripts/strips_probe.py heat float32 16384 100 > $O/strips_heat.txt 2>&1
head -12 $O/strips_heat.txt; tail -7 $O/strips_heat.txt
timeout 900 python -m pytest tests/test_multirank_gpu.py -x -q > $O/pytest_multirank.log 2>&1; echo "rc=$?" >> $O/pytest_multirank.log
tail -3 $O/pytest_multirank.log
