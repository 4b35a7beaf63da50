#!/usr/bin/env bash
# Final evidence after the grid-balance and ring-depth changes: full GPU suite,
# smoke, bench line, reference arm, bench launch list at the headline block,
# ncu of heat 16384^2 48x8 (one block, three-stage ring) and the config-4 oracle block.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r04z}; mkdir -p $O
timeout 2000 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; rc=$?
echo "pytest rc=$rc" | tee -a $O/pytest_gpu.log; tail -4 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -c 400 $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_32x28.csv \
  python bench.py --steps 2 --warmup 3 --wc 32 --wr 28 --no-e2e --no-cpu --no-temporal > /dev/null 2>&1; echo "launches rc=$?"
OUT=${1:-r04z} bash scripts/r02_ncu_vec.sh \
  "heat_48x8_post k_stencil_tma heat float32 16384 16384 48 8 4 auto nearest" \
  "box_16x8_final k_stencil_tma boxmean float32 4096 4096 16 8 4 auto nearest" > /dev/null 2>&1
rm -f $O/*_source.csv
ls $O
