#!/usr/bin/env bash
# Heat 16384^2 vector-path sizes (48x8 slow, 54x8 fast, 52x8 slow, scalar 88x8 best):
# ncu --set full of each, then the default bench line (grid balance in) and the
# bench launch list at the bench's tuned block.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r04h}; mkdir -p $O
OUT=${1:-r04h} bash scripts/r02_ncu_vec.sh \
  "heat_48x8 k_stencil_tma heat float32 16384 16384 48 8 4 auto nearest" \
  "heat_54x8 k_stencil_tma heat float32 16384 16384 54 8 4 auto nearest" \
  "heat_52x8 k_stencil_tma heat float32 16384 16384 52 8 4 auto nearest" \
  "heat_88x8 k_stencil_tma heat float32 16384 16384 88 8 4 auto nearest" > /dev/null 2>&1
rm -f $O/*_source.csv
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -c 400 $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_32x28.csv \
  python bench.py --steps 2 --warmup 3 --wc 32 --wr 28 --no-e2e --no-cpu --no-temporal > /dev/null 2>&1; echo "launches rc=$?"
ls $O
