#!/usr/bin/env bash
# Round-2 (late) check: online-tuning tests, ncu of the config-4 kernel at its
# oracle block with the source page, then the default bench line.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r03c}; mkdir -p $O
timeout 600 python -m pytest tests/test_online_tuning.py -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest.log
tail -5 $O/pytest.log
OUT=${1:-r03c} bash scripts/r02_ncu_vec.sh "box_16x8 k_stencil_tma boxmean float32 4096 4096 16 8 4 auto nearest" > /dev/null 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -c 800 $O/bench.err
