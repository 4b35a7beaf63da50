#!/usr/bin/env bash
# Retrain the committed forest bundles from the layered study data: round 1's
# samples (the synthetic kernels) under the real kernels' 30-observation
# re-sweep in ${REAL:-results/b200/real30} (later layers replace whole
# scenarios): model.json on every scenario, model_loko_{gol,he}.json without
# any scenario of that kernel (the bench's held-out check).
set -euo pipefail
cd "$(dirname "$0")/.."
B=results/b200
REAL=${REAL:-$B/real30}
T=$(mktemp -d)
zcat $B/samples.csv.gz > $T/r1_samples.csv
cp $B/refused.csv $T/r1_refused.csv
cp $B/contexts.csv $T/r1_contexts.csv
for f in samples refused contexts; do xz -dc $REAL/${f}_real30.csv.xz > $T/r2_$f.csv; done
LAYERS="--samples $T/r1_samples.csv --refused $T/r1_refused.csv --contexts $T/r1_contexts.csv \
        --samples $T/r2_samples.csv --refused $T/r2_refused.csv --contexts $T/r2_contexts.csv"
BIN=paper_1511_02490_b200/lib/wgtb
$BIN train --scenarios $B/descriptors $LAYERS --technique forest-nn --out $B/model.json
KERNELS=$(ls $B/descriptors/kernels | sed 's/\.json$//')
for held in gol he; do
  keep=""
  for k in $KERNELS; do [ "$k" != "$held" ] && keep="$keep --kernel $k"; done
  $BIN train --scenarios $B/descriptors $LAYERS $keep --technique forest-nn --out $B/model_loko_$held.json
done
rm -rf $T
