#!/usr/bin/env bash
# Exhaustive wc x wr sweep on the B200 for the autotuning study (BASELINE
# config 5): the 40 synthetic kernels of generate_kernels(40, 17) + the 6
# reference kernels x the descriptor datasets (results/b200/descriptors; pass
# --dataset / --kernel filters through to `wgtb collect`).  Resumable: completed scenarios in results/b200 are
# kept.  Output lands in gpurun_out/b200 (copy back into results/b200).
set -euo pipefail
cd "$(dirname "$0")/.."
BIN=paper_1511_02490_b200/lib/wgtb
OUT=gpurun_out/b200
mkdir -p "$OUT"
[ -d results/b200/descriptors ] || { echo "missing results/b200/descriptors"; exit 2; }
cp -r results/b200/descriptors "$OUT/" 2>/dev/null || true
for f in samples.csv refused.csv contexts.csv; do
  [ -f results/b200/$f ] && cp results/b200/$f "$OUT/$f"
done
$BIN features > "$OUT/device.json"
timeout "${SWEEP_SECONDS:-3000}" $BIN collect --scenarios results/b200/descriptors --out "$OUT/samples.csv" \
  --refused "$OUT/refused.csv" --contexts "$OUT/contexts.csv" --samples "${SAMPLES:-5}" --warmup 2 --store mean --resume "$@" \
  2> "$OUT/collect.log" || echo "collect stopped (rc=$?)"
tail -3 "$OUT/collect.log"
wc -l "$OUT/contexts.csv"
# gpurun copies back at most 64 MiB: ship the samples compressed
gzip -f "$OUT/samples.csv"
rm -rf "$OUT/descriptors"
