#!/usr/bin/env bash
# Executable synthetic kernels for the autotuning study:
# `wgtb gen-kernel` applies the paper's template substitution (PAPER.md:
# 206-222) to every synthetic descriptor of the study (generate_kernels(40,
# 17)), then results/generated/Makefile compiles each functor into the
# executor's kernel templates (lib/lib<name>.so) and its C reference
# (lib/lib<name>_ref.so).  Generated sources are build outputs (git-ignored):
# they are a pure function of the committed descriptors.
set -euo pipefail
cd "$(dirname "$0")/.."
W=paper_1511_02490_b200/lib/wgtb
mkdir -p results/generated/src
for k in results/b200/descriptors/kernels/synthetic-*.json; do
  n=$(basename "$k" .json)
  [ -f "results/generated/src/$n.cu" ] || $W gen-kernel --kernel-json "$k" --out results/generated/src > /dev/null
done
make -s -C results/generated -j"$(nproc)"
ls results/generated/lib | wc -l
