#!/usr/bin/env bash
cd "$(dirname "$0")/.."
O=gpurun_out/c30; mkdir -p $O
timeout 600 python -m pytest tests/test_gol_bits.py -x -q > $O/pytest_bits.log 2>&1; echo "rc=$?" >> $O/pytest_bits.log; tail -2 $O/pytest_bits.log
timeout 900 python scripts/bits_probe.py > $O/bits_probe.txt 2>&1; head -8 $O/bits_probe.txt
for k in fused; do
  timeout 300 compute-sanitizer --tool racecheck --racecheck-report hazard python scripts/sanitize_temporal.py $k >> $O/sanitizer_racecheck.log 2>&1
  timeout 300 compute-sanitizer --tool memcheck python scripts/sanitize_temporal.py $k >> $O/sanitizer_memcheck.log 2>&1
done
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ran " $O/sanitizer_*.log
