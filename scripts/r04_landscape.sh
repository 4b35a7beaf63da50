#!/usr/bin/env bash
# Deep-ring policy A/B over a slice of the space (two rounds, alternating), + L2 promotion 128 vs 256.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r04l}; mkdir -p $O
timeout 300 python -m pytest tests/test_stencil_parity.py -k "balanced_grid or heat or boxmean" -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest.log
for r in 1 2; do
  SK_DEEP_RING=0 timeout 900 python scripts/landscape_probe.py 7 >> $O/land.jsonl 2>> $O/land.err
  timeout 900 python scripts/landscape_probe.py 7 >> $O/land.jsonl 2>> $O/land.err
  SK_L2_PROMO=128 timeout 900 python scripts/landscape_probe.py 7 >> $O/land.jsonl 2>> $O/land.err
done
wc -l $O/land.jsonl
