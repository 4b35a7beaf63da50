#!/usr/bin/env bash
# Resumable GPU sweep of the 40 generated synthetic kernels (scripts/sweep_generated.py):
# partial results live compressed in results/generated_r02/ (gpurun_out does not travel).
set -uo pipefail
cd "$(dirname "$0")/.."
O=gpurun_out/gen_r02; R=results/generated_r02; mkdir -p $O $R
for f in samples.csv refused.csv contexts.csv collect.log; do
  [ -f $R/$f.xz ] && xz -dc $R/$f.xz > $O/$f
done
[ -d results/generated/lib ] || bash scripts/gen_study_kernels.sh
timeout "${SWEEP_SECONDS:-2400}" python scripts/sweep_generated.py $O 5 "${BUDGET:-2100}"
echo "sweep rc=$?"
wc -l $O/contexts.csv
for f in samples.csv refused.csv contexts.csv collect.log; do xz -T0 -6 -f $O/$f; done
ls -la $O
