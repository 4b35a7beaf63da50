#!/usr/bin/env bash
# Round-2 bench evidence: the default bench line, the reference arm, and the
# ncu launch list of a short bench run (the roofline's launch share).
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r02bench}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -c 1500 $O/bench.err
timeout 900 python bench.py --impl reference --steps 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-temporal --no-configs > $O/ncu_bench.log 2>&1; echo "ncu rc=$?"
