#!/usr/bin/env bash
# Bit-plane GoL: parity tests, the (TB, wc, wr, K) probe and, with PROFILE set
# ("tb wc wr k reps"), one ncu --set full capture of a middle (bits->bits) launch.
cd "$(dirname "$0")/.."
O=gpurun_out/bits1; mkdir -p $O
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests/test_gol_bits.py -q -x > $O/pytest_bits.log 2>&1; echo "rc=$?" >> $O/pytest_bits.log
  tail -3 $O/pytest_bits.log
fi
if [ -z "$NOPROBE" ]; then
  timeout 1200 python scripts/bits_probe.py > $O/bits_probe.txt 2>&1
  head -12 $O/bits_probe.txt; tail -9 $O/bits_probe.txt
fi
if [ -n "$PROFILE" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gol_strips -s 1 -c 1 -o $O/prof_$(echo $PROFILE | tr ' ' '_') python scripts/profile_bits.py 8192 $PROFILE > $O/ncu.log 2>&1
  tail -2 $O/ncu.log
fi
