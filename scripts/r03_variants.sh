#!/usr/bin/env bash
# A/B of kernel variants built under variants/<name>/ (not committed): the
# config-4 probe for each, round-robin twice.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r03v}; mkdir -p $O
for rep in 1 2; do
  for v in ${VARIANTS:-v0 vA vB main}; do
    if [ $v = main ]; then VR=""; else VR=$PWD/variants/$v; fi
    VARIANT_ROOT=$VR QUICK=1 timeout 300 python scripts/box_probe.py 30 > $O/probe_${v}_$rep.json 2> $O/probe_${v}_$rep.err
    echo "$v $rep rc=$?"
  done
done
