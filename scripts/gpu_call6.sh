#!/usr/bin/env bash
cd "$(dirname "$0")/.."
O=gpurun_out/c7; mkdir -p $O
timeout 300 python -m pytest tests/test_peer_halo.py -x -q > $O/pytest_peer.log 2>&1; echo "rc=$?" >> $O/pytest_peer.log
tail -3 $O/pytest_peer.log
timeout 600 python -m pytest tests/test_cross_strips.py -x -q > $O/pytest_strips.log 2>&1; echo "rc=$?" >> $O/pytest_strips.log
tail -3 $O/pytest_strips.log
timeout 900 python scripts/strips_probe.py heat float32 16384 100 6,8,10,12 > $O/strips_heat.txt 2>&1
head -14 $O/strips_heat.txt; tail -6 $O/strips_heat.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cross_strips -s 1 -c 1 \
  -o $O/prof_strips_heat_tb8_k8_32x12 python scripts/profile_strips.py 16384 8 8 32 12 1 > $O/ncu_full.log 2>&1
tail -1 $O/ncu_full.log
