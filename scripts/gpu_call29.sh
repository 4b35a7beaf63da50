#!/usr/bin/env bash
cd "$(dirname "$0")/.."
O=gpurun_out/c29; mkdir -p $O
timeout 600 python -m pytest tests/test_stencil_parity.py -q -k "special_values" > $O/pytest_special.log 2>&1; echo "rc=$?" >> $O/pytest_special.log; tail -2 $O/pytest_special.log
timeout 900 paper_1511_02490_b200/lib/wgtb collect --scenarios results/config4/descriptors --out $O/config4_samples.csv \
  --refused $O/config4_refused.csv --contexts $O/config4_contexts.csv --samples 30 --warmup 3 --store mean \
  > $O/config4.log 2>&1; echo "config4 rc=$?"; tail -2 $O/config4.log
for k in strips bitplane fused peer streamed; do
  timeout 300 compute-sanitizer --tool racecheck --racecheck-report hazard python scripts/sanitize_temporal.py $k >> $O/sanitizer_racecheck.log 2>&1
  timeout 300 compute-sanitizer --tool memcheck python scripts/sanitize_temporal.py $k >> $O/sanitizer_memcheck.log 2>&1
done
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ran " $O/sanitizer_*.log
