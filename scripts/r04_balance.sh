#!/usr/bin/env bash
# Grid-balance A/B (SK_GRID_BALANCE=0 vs default) + its parity test.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r04b}; mkdir -p $O
timeout 600 python -m pytest tests/test_stencil_parity.py -k "balanced_grid or boxmean or heat" -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest.log; tail -3 $O/pytest.log
for r in 1 2; do
  SK_GRID_BALANCE=0 timeout 600 python scripts/grid_balance_probe.py 15 >> $O/probe.jsonl 2> $O/probe0.err
  timeout 600 python scripts/grid_balance_probe.py 15 >> $O/probe.jsonl 2> $O/probe1.err
done
cat $O/probe.jsonl
