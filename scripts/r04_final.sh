#!/usr/bin/env bash
# Final round-2 evidence on the current build: full GPU suite, smoke, the default
# bench line, the reference arm, the bench launch list, and ncu --set full of the
# config-4 kernel after the K=8/80-register change (post-change digest).
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r04f}; mkdir -p $O
timeout 2000 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; rc=$?
echo "pytest rc=$rc" | tee -a $O/pytest_gpu.log; tail -6 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -c 600 $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-temporal > /dev/null 2>&1; echo "launches rc=$?"
OUT=${1:-r04f} bash scripts/r02_ncu_vec.sh "box_16x8_post k_stencil_tma boxmean float32 4096 4096 16 8 4 auto nearest" > /dev/null 2>&1
ls $O
