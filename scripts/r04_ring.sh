#!/usr/bin/env bash
# Ring depth A/B: default policy vs lag 1 (prefetch stages-1 tiles), min 3/4 stages (fewer, deeper CTAs).
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r04r}; mkdir -p $O
timeout 300 python -m pytest tests/test_stencil_parity.py -k "balanced_grid" -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest.log
for r in 1 2; do
  for cfg in "" "SK_RING_LAG=1" "SK_MIN_STAGES=3" "SK_MIN_STAGES=3 SK_RING_LAG=1" "SK_MIN_STAGES=4 SK_RING_LAG=1" "SK_MIN_STAGES=4"; do
    echo "{\"cfg\": \"$cfg\"}" >> $O/probe.jsonl
    env $cfg SK_L2_PROMO=128 timeout 600 python scripts/l2_promo_probe.py 11 >> $O/probe.jsonl 2>> $O/probe.err
  done
done
cat $O/probe.jsonl
