#!/usr/bin/env bash
# Peer exchange + strips tests, strip-kernel ncu capture, heat and gol bench lines.
cd "$(dirname "$0")/.."
O=gpurun_out/c5; mkdir -p $O
timeout 300 python -m pytest tests/test_peer_halo.py -x -q > $O/pytest_peer.log 2>&1; echo "rc=$?" >> $O/pytest_peer.log
tail -3 $O/pytest_peer.log
timeout 600 python -m pytest tests/test_cross_strips.py -x -q > $O/pytest_strips.log 2>&1; echo "rc=$?" >> $O/pytest_strips.log
tail -3 $O/pytest_strips.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cross_strips -s 1 -c 1 \
  -o $O/prof_strips_heat_tb8_k8_32x12 python scripts/profile_strips.py 16384 8 8 32 12 1 > $O/ncu_full.log 2>&1
tail -1 $O/ncu_full.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches_strips.csv python scripts/profile_strips.py 16384 8 8 32 12 1 > $O/ncu_list.log 2>&1
timeout 900 python bench.py --config heat --steps 5 > $O/bench_heat.json 2> $O/bench_heat.err; echo "bench heat rc=$?"
cat $O/bench_heat.json
timeout 900 python bench.py > $O/bench_gol.json 2> $O/bench_gol.err; echo "bench gol rc=$?"
cat $O/bench_gol.json
