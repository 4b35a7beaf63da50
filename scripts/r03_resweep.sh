#!/usr/bin/env bash
# Round-2 (late) re-sweep with the current executor (AUTO = vector work-items where
# they fit): the six reference kernels + the BASELINE configs' five_point and
# boxmean (5,1,3,0) x all datasets, 30 observations per
# size stored one line per observation (no means), 3 warm-ups, L2 scrubbed
# before every sample; and the config-4 scenario (boxmean 5,1,3,0 4096^2).
# Fresh sweep (the executor's AUTO path choice changed after the first re-sweep:
# vector work-items only within the vector kernel's thread bound, packed box mean).
# Resumable (--resume) within the call; outputs under gpurun_out/resweep3.
set -uo pipefail
cd "$(dirname "$0")/.."
BIN=paper_1511_02490_b200/lib/wgtb
O=gpurun_out/resweep3; mkdir -p $O
if [ "${CONFIG4:-1}" = 1 ]; then
  timeout 900 $BIN collect --scenarios results/config4/descriptors --out $O/config4_samples.csv \
    --refused $O/config4_refused.csv --contexts $O/config4_contexts.csv --samples 30 --warmup 3 \
    --store all 2> $O/config4_collect.log
  echo "config4 rc=$?"
fi
timeout "${SWEEP_SECONDS:-2400}" $BIN collect --scenarios results/b200/descriptors \
  --kernel gaussian --kernel gol --kernel he --kernel nms --kernel sobel --kernel threshold \
  --kernel five_point --kernel boxmean-5130 \
  --out $O/samples_real30.csv --refused $O/refused_real30.csv --contexts $O/contexts_real30.csv \
  --samples 30 --warmup 3 --store all --resume 2>> $O/real30_collect.log
echo "real30 rc=$?"
tail -2 $O/real30_collect.log
wc -l $O/contexts_real30.csv
# the copy-back is capped at 64 MiB: ship compressed
for f in samples_real30.csv refused_real30.csv contexts_real30.csv config4_samples.csv; do
  [ -f $O/$f ] && xz -T0 -6 -f $O/$f
done
ls -la $O
