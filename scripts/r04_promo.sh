#!/usr/bin/env bash
# L2 promotion A/B (two rounds, round-robin over the settings) + ncu DRAM bytes of heat 48x8 at 128 B.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r04p}; mkdir -p $O
for r in 1 2; do for p in 256 128 64 0; do
  SK_L2_PROMO=$p timeout 600 python scripts/l2_promo_probe.py 15 >> $O/probe.jsonl 2>> $O/probe.err
done; done
cat $O/probe.jsonl
