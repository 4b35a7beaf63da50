#!/usr/bin/env bash
cd "$(dirname "$0")/.."
O=gpurun_out/c14; mkdir -p $O
timeout 900 python bench.py --config heat --steps 10 > $O/bench_heat.json 2> $O/bench_heat.err; echo "bench heat rc=$?"
cat $O/bench_heat.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_gol_bench.csv \
  python bench.py --steps 2 --warmup 3 --wc 128 --wr 8 --no-e2e --no-cpu --no-temporal > $O/bench_under_ncu.log 2>&1
echo "ncu rc=$?"; wc -l $O/launches_gol_bench.csv
