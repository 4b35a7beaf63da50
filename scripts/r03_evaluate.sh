#!/usr/bin/env bash
# The study on the layered data (round 1's samples under the real kernels'
# re-sweep in ${REAL:-results/b200/real30}): all 14 techniques, 10-fold and
# leave-one-kernel-out, with the human-expert comparison and the 10-fold rows.
# usage: scripts/r03_evaluate.sh [OUT_PREFIX]
set -euo pipefail
cd "$(dirname "$0")/.."
B=results/b200
REAL=${REAL:-$B/real30}
OUT=${1:-$B/evaluate_r03}
T=$(mktemp -d)
zcat $B/samples.csv.gz > $T/r1_samples.csv
for f in samples refused contexts; do xz -dc $REAL/${f}_real30.csv.xz > $T/r2_$f.csv; done
LAYERS="--samples $T/r1_samples.csv --refused $B/refused.csv --contexts $B/contexts.csv \
        --samples $T/r2_samples.csv --refused $T/r2_refused.csv --contexts $T/r2_contexts.csv"
BIN=paper_1511_02490_b200/lib/wgtb
for part in kfold loo-kernel; do
  extra=""
  [ $part = kfold ] && extra="--metrics $T/metrics.csv"
  $BIN evaluate --scenarios $B/descriptors $LAYERS --technique all --partition $part --expert $extra \
    > ${OUT}_$part.txt
done
xz -T0 -6 -c $T/metrics.csv > $B/metrics_r03_kfold.csv.xz
rm -rf $T
